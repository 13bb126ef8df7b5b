# throughput of the reference-layout (AoS, m_pad 16) path vs the native AoSoA path
exec > gpurun_out/aos.log 2>&1
python - <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_2003_12787_b200 as S
for n, E in ((8, 32768), (6, 32768), (10, 8192), (9, 8192)):
    q, par = S.generate(0, 1, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=9)
    qa = torch.empty(E, n ** 3 * 16, dtype=torch.float64, device='cuda')
    S.convert_layout(n, 9, E, S.LAYOUT_AOSOA, 9, q, S.LAYOUT_AOS, 16, qa)
    for layout, x, st in ((S.LAYOUT_AOSOA, q, 9), (S.LAYOUT_AOS, qa, 16)):
        plan = S.Plan(n, S.elastic_pde(), layout=layout, q_stride=st, out_stride=st, par_kind=S.PAR_RHO_CP_CS)
        out = plan.alloc_output(E)
        for _ in range(3): plan.predict(x, 1e-3, par=par, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): plan.predict(x, 1e-3, par=par, out=out)
        e1.record(); torch.cuda.synchronize()
        print(n, 'AoSoA' if layout == S.LAYOUT_AOSOA else 'AoS16', E / (e0.elapsed_time(e1) / 10 * 1e-3))
PY
# kernel-level breakdown of the AoS path at nDof 8 (ncu launch durations and DRAM bytes)
cat > /tmp/aos8.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_2003_12787_b200 as S
n, E = 8, 32768
q, par = S.generate(0, 1, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=9)
qa = torch.empty(E, n ** 3 * 16, dtype=torch.float64, device='cuda')
S.convert_layout(n, 9, E, S.LAYOUT_AOSOA, 9, q, S.LAYOUT_AOS, 16, qa)
plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOS, q_stride=16, out_stride=16, par_kind=S.PAR_RHO_CP_CS)
out = plan.alloc_output(E)
for _ in range(3): plan.predict(qa, 1e-3, par=par, out=out)
torch.cuda.synchronize()
PY
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python /tmp/aos8.py 2>/dev/null | \
  awk -F'","' 'NF>6{print $5, $(NF-2), $(NF-1), $NF}' | tail -24

#!/usr/bin/env python3
"""Benchmark of the B200 linear ADER-DG Space-Time Predictor (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c1..c5]

A "step" is one pass of the STP (CK recursion + favg + 12 face arrays) over one batch of
synthetic elastic elements.  Default workload: BASELINE config C3 -- order N=7 (nDof 8),
131,072 elements per GPU, padded AoSoA input with nVar padded to 12, per-element random
material.  Under torchrun (N > 1) every rank owns a contiguous element range (weak scaling for
c1-c4, strong scaling for c5) with no collective on the hot path; NCCL only reduces the max
step time and a checksum after timing.

`value` is device-resident throughput (inputs in HBM, CUDA events, max over ranks);
`e2e` is the same metric through the public host-buffer API (aderstp_predict_batch_host) with
pinned host inputs and outputs, copies inside the timed region.  `--impl reference` times the
reference's own CPU implementation (oracle/_ref = the unmodified reference sources compiled by
oracle/Makefile) on the host cores over a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# the host cores this process may use, read before any OpenMP runtime binds the main thread
try:
    HOST_CORES = len(os.sched_getaffinity(0))
except AttributeError:
    HOST_CORES = os.cpu_count() or 1



def _load_shard_module():
    """paper_2003_12787_b200/shard.py loaded as a standalone module: importing it through the
    package would run the package __init__, which maps libaderstp.so -- and the reference arm's
    process must never load our library (it times the unmodified reference only)."""
    import importlib.util
    path = os.path.join(ROOT, "paper_2003_12787_b200", "shard.py")
    spec = importlib.util.spec_from_file_location("_aderstp_bench_shard", path)
    mod = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = mod
    spec.loader.exec_module(mod)
    return mod


_shard = _load_shard_module()
barrier, chunks, env_world = _shard.barrier, _shard.chunks, _shard.env_world
max_over_ranks, sum_over_ranks = _shard.max_over_ranks, _shard.sum_over_ranks
strong_shard, weak_shard = _shard.strong_shard, _shard.weak_shard

METRIC = "linear STP elements/s & fp64 GFLOP/s (% of roofline) vs order N, 1–8 B200"
UNIT = "elements/s"

# BASELINE.json configs (order N = polynomial degree, nDof = N+1)
CONFIGS = {
    "c1": dict(n=4, elems=64, dist=0, q_stride=9,
               desc="C1: elastic STP order N=3 (nDof 4), 64 elements, Q~U[-1,1]"),
    "c2": dict(n=6, elems=32768, dist=2, q_stride=9,
               desc="C2: elastic STP order N=5 (nDof 6), 32,768 elements (32^3 periodic grid), "
                    "Q = 3 random-phase sinusoids per quantity"),
    "c3": dict(n=8, elems=131072, dist=0, q_stride=12,
               desc="C3: elastic STP order N=7 (nDof 8), 131,072 elements/GPU, padded AoSoA "
                    "(nVar padded to 12), Q~U[-1,1], per-element random material"),
    "c4": dict(n=10, elems=65536, dist=1, q_stride=9,
               desc="C4: elastic STP order N=9 (nDof 10), 65,536 elements, Q~N(0,1)"),
    # order N=3 (nDof 4) as a large batch: not a BASELINE config (C1 has 64 elements); the
    # warp-per-element kernel stp_wpe takes nDof 4 batches of >= 16,384 elements
    "n4": dict(n=4, elems=131072, dist=0, q_stride=9,
               desc="elastic STP order N=3 (nDof 4), 131,072 elements, Q~U[-1,1] (kernel stp_wpe)"),
    # order N=8 (nDof 9): not a BASELINE config, measured because north_star's >=50% target covers
    # every order >= 7
    "n9": dict(n=9, elems=65536, dist=1, q_stride=9,
               desc="elastic STP order N=8 (nDof 9), 65,536 elements, Q~N(0,1)"),
    # C5: 1,048,576 elements split evenly over the GPUs (strong scaling); a GPU streams its shard
    # through fixed-size launches (inputs resident in HBM, output buffers reused per launch)
    "c5": dict(n=8, elems=1048576, dist=0, q_stride=9, strong=True, chunk=131072,
               desc="C5: elastic STP order N=7 (nDof 8), 1,048,576 elements split over the GPUs"),
    "c5n6": dict(n=6, elems=1048576, dist=0, q_stride=9, strong=True, chunk=262144,
                 desc="C5: elastic STP order N=5 (nDof 6), 1,048,576 elements split over the GPUs"),
}
SEED = 20031278
# dt of every config: stable_dt (proj/src/solver.cpp:170-174) at CFL 0.5 for the material's largest
# P-wave speed (cp ~ U[4,6] per element, so cp <= 6).  A fixed bound instead of the sampled maximum
# keeps dt identical across both bench arms, every GPU count and every sample size.
CFL, CP_BOUND = 0.5, 6.0
# elements timed per step by the CPU reference (C1/C2 the full set, C3-C5 a
# fixed 16,384-element subset -- elements 0..16,383 of the same seeded workload)
REFERENCE_SAMPLE = {"c1": 64, "n4": 16384, "c2": 32768, "c3": 16384, "c4": 16384, "n9": 16384, "c5": 16384, "c5n6": 16384}
REFERENCE_REPS = 3


def config_dt(n):
    return CFL / (3.0 * CP_BOUND * (2.0 * n - 1.0))


def config_of(name, world):
    """The workload description both arms print (identical keys and values for one --config and
    --gpus); what a run did beyond the workload (launches, graphs, samples) goes elsewhere."""
    cfg = CONFIGS[name]
    n = cfg["n"]
    total = cfg["elems"] if cfg.get("strong") else world * cfg["elems"]
    return {"workload": cfg["desc"], "name": name, "order": n - 1, "n_dof": n, "quantities": 9,
            "global_elements": total, "elements_per_gpu": total // world if cfg.get("strong") else cfg["elems"],
            "layout": f"AoSoA [e][k3][k2][s<{cfg['q_stride']}][k1] in, [e][k3][k2][9][k1] out",
            "input_distribution": ["U[-1,1]", "N(0,1)", "3 random-phase sinusoids"][cfg["dist"]],
            "material": "per element rho~U[2,3], cp~U[4,6], cs~U[2,3.5]",
            "dt": config_dt(n), "cfl": CFL, "seed": SEED,
            "parallelism": f"element shards x{world} (no hot-path collective)",
            "l2": "no flush needed: inputs %.2f GB and outputs %.2f GB per GPU step vs 126 MB L2" % (
                (total // world if cfg.get("strong") else cfg["elems"]) * n ** 3 * cfg["q_stride"] * 8 / 1e9,
                (total // world if cfg.get("strong") else cfg["elems"]) * (4 * n ** 3 * 9 + 12 * n * n * 9) * 8 / 1e9)}


def fp64_peak():
    """fp64 pipe peak of this pool's B200, measured (MEASURED_PEAKS.json has no fp64 entry):
    profiles/fp64_peaks_r02.json, written by tools/fp64_peaks.py -- DMMA m8n8k4 f64 sustained over
    seconds with the SM clock and throttle reasons sampled beside it (DFMA alone is lower; the
    larger of the two pipes is the denominator).  Returns (FLOP/s, source description)."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peaks_r02.json")) as f:
            d = json.load(f)
        tf = max(d["dmma_sustained_tflops"], d["dfma_sustained_tflops"])
        ck = d["dmma_sustained_clocks"]
        return tf * 1e12, (f"measured sustained DMMA fp64 {tf} TFLOP/s at SM {ck['sm_mhz_median']} MHz "
                           f"(reasons {ck['reasons'] or 'none'}), profiles/fp64_peaks_r02.json")
    except (OSError, KeyError, ValueError):
        return 37.1e12, "measured DMMA fp64 37.1 TFLOP/s, profiles/fp64_peaks_r01.txt (no clock record)"


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]) * 1e9, "MEASURED_PEAKS.json hbm_gbs (measured)"
    except Exception:
        return 6.65e12, "fallback 6.65 TB/s (B200_PROFILING.md)"


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, device_index):
        self.samples, self.reasons, self.ok = [], 0, False
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            uuid = str(torch.cuda.get_device_properties(device_index).uuid)
            try:
                self.h = pynvml.nvmlDeviceGetHandleByUUID("GPU-" + uuid)
            except Exception:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        names = [n for bit, n in self.REASONS.items() if self.reasons & bit]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


def dist_setup():
    import torch
    world, rank, local = env_world()
    if world > 1:
        import torch.distributed as dist
        # ADERSTP_BENCH_BACKEND=gloo validates the multi-rank flow on a box with fewer GPUs than
        # ranks (ranks then share devices; never a timing run).  Default: NCCL, one GPU per rank.
        backend = os.environ.get("ADERSTP_BENCH_BACKEND", "nccl")
        local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def load_ncu_field(cfg_name, key):
    """A field of the committed ncu summary (profiles/ncu_summary.json) for this config."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f).get(cfg_name, {}).get(key)
    except Exception:
        return None


def load_traffic(cfg_name, elements_per_launch):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the STP kernel, from the
    committed ncu --set full capture (profiles/ncu_summary.json, measured per element and scaled
    to this run's launch size)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            per = json.load(f).get(cfg_name, {}).get("dram_bytes_per_element")
        return None if per is None else per * elements_per_launch
    except Exception:
        return None


def shard_of(cfg, world, rank):
    if cfg.get("strong"):
        return strong_shard(cfg["elems"], world, rank)
    return weak_shard(cfg["elems"], world, rank)


def make_plan(S, cfg):
    return S.Plan(cfg["n"], S.elastic_pde(), layout=S.LAYOUT_AOSOA, q_stride=cfg["q_stride"], out_stride=9,
                  par_kind=S.PAR_RHO_CP_CS, check_inputs=True)


def measure_device(S, cfg, world, rank, steps, warmup, want_clocks=True):
    """Device-resident timing of one config on this rank's shard (max over ranks)."""
    import torch
    n = cfg["n"]
    sh = shard_of(cfg, world, rank)
    grid = round(cfg["elems"] ** (1.0 / 3.0)) if cfg["dist"] == 2 else 1
    q, par = S.generate(cfg["dist"], SEED, n, sh.start, sh.count, grid=grid, layout=S.LAYOUT_AOSOA,
                        q_stride=cfg["q_stride"])
    dt = config_dt(n)
    plan = make_plan(S, cfg)
    chunk = max(1, min(cfg.get("chunk", sh.count), sh.count))
    out = plan.alloc_output(chunk)
    ranges = [(s0 - sh.start, c) for s0, c in chunks(sh, chunk)]

    def step():
        for off, c in ranges:
            o = S.PredictorOutput(out.qavg[:c], out.favg[:c], out.face_q[:c], out.face_f[:c])
            plan.predict(q[off:off + c], dt, par=par[off:off + c], out=o)

    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        step()
    plan.status()
    torch.cuda.synchronize()
    # one step (all its launches) captured once in a CUDA graph and replayed: the small configs
    # (C1: a 10 us kernel) are otherwise bound by the host-side launch path, not the GPU
    run, graphed = step, False
    try:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        graph.replay()
        torch.cuda.synchronize()
        run, graphed = graph.replay, True
    except Exception:  # noqa: BLE001 (fall back to direct launches)
        torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(torch.cuda.current_device()) if want_clocks else None
    barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.__enter__()
    ev0.record(stream)
    for _ in range(steps):
        run()
    ev1.record(stream)
    torch.cuda.synchronize()
    if sampler:
        sampler.__exit__()
    barrier()
    ms = ev0.elapsed_time(ev1) / steps
    plan.status()
    checksum = float(out.qavg.sum().item()) + float(out.face_q.sum().item())
    res = dict(ms=max_over_ranks(ms, device="cuda"), dt=dt,
               checksum=sum_over_ranks(checksum, device="cuda"),
               clocks=sampler.summary() if sampler else None, plan=plan, shard=sh,
               launches_per_step=len(ranges), elements_per_launch=chunk, cuda_graph=graphed)
    del q, par, out
    return res


def measure_reference_layout(S, cfg, steps, warmup):
    """The drop-in boundary on the reference's own element layout: C3's workload (nDof 8,
    131,072 elements, per-element material) held as ElementTensor AoS rows (quantity padded to
    m_pad = 16, proj/src/layout.cpp:9-21) in and PredictorOutput AoS rows out.  Device-resident,
    CUDA events; at nDof 8 the tuned kernel reads and writes the node rows itself."""
    import torch
    n, E = cfg["n"], cfg["elems"]
    q9, par = S.generate(cfg["dist"], SEED, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=9)
    q = torch.empty(E, n ** 3 * 16, dtype=torch.float64, device="cuda")
    S.convert_layout(n, 9, E, S.LAYOUT_AOSOA, 9, q9, S.LAYOUT_AOS, 16, q)
    del q9
    plan = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOS, q_stride=16, out_stride=16, par_kind=S.PAR_RHO_CP_CS)
    out = plan.alloc_output(E)
    dt = config_dt(n)
    for _ in range(warmup):
        plan.predict(q, dt, par=par, out=out)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(steps):
        plan.predict(q, dt, par=par, out=out)
    ev1.record(stream)
    torch.cuda.synchronize()
    plan.status()
    ms = ev0.elapsed_time(ev1) / steps
    del q, out
    return {"workload": "C3 on the reference layout: ElementTensor AoS (m_pad 16) in, PredictorOutput AoS out",
            "elements_per_s": E / (ms * 1e-3), "ms_per_step": ms,
            "path": "stp_dmma8<AOS>: planes staged from the node rows, qavg/favg written as node rows"}


def measure_table_pde(S, steps, warmup, n=8, E=65536):
    """The user-LinearPde path: the reference's advection system with m = 8 quantities
    (proj/src/pde.cpp:61-85), device-resident -- at nDof 8 on the tensor cores (stp_dmma8_table),
    at nDof 9 / 10 on the line-pass table kernel (stp_tlp)."""
    import torch
    m = 8
    pde = S.advection_pde((1.0, 0.5, 0.25), m)
    g = torch.Generator(device="cuda").manual_seed(SEED)
    q = torch.rand(E, n ** 3 * m, dtype=torch.float64, device="cuda", generator=g) * 2.0 - 1.0
    plan = S.Plan(n, pde, layout=S.LAYOUT_AOSOA, q_stride=m, out_stride=m)
    out = plan.alloc_output(E)
    dt = 0.5 / (3.0 * 1.0 * (2 * n - 1))
    for _ in range(warmup):
        plan.predict(q, dt, out=out)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(steps):
        plan.predict(q, dt, out=out)
    ev1.record(stream)
    torch.cuda.synchronize()
    plan.status()
    ms = ev0.elapsed_time(ev1) / steps
    del q, out
    return {"workload": f"advection PDE, m = 8 quantities, nDof {n}, {E:,} elements, Q~U[-1,1] (user LinearPde path)",
            "elements_per_s": E / (ms * 1e-3), "ms_per_step": ms,
            "kernel": "stp_dmma8_table" if n == 8 else "stp_tlp" if n >= 9 else "stp_dmmat / stp_kernel"}


def measure_general_pde(S, steps, warmup, m=21, n=8, E=16384):
    """A dense user LinearPde (every A_d and B_d entry nonzero; m = 21 is the paper's application
    size) at nDof 8, device-resident: the tensor-core kernel stp_gdense.cu (the scalar general
    kernel stp_general.cu with ADERSTP_NO_GDENSE=1)."""
    import numpy as np
    import torch
    rng = np.random.default_rng(SEED)
    A = [rng.uniform(-1, 1, (m, m)) / m ** 0.5 for _ in range(3)]
    B = [rng.uniform(-0.5, 0.5, (m, m)) / m ** 0.5 for _ in range(3)]
    pde = S.linear_pde(A, B)
    g = torch.Generator(device="cuda").manual_seed(SEED)
    q = torch.rand(E, n ** 3 * m, dtype=torch.float64, device="cuda", generator=g) * 2.0 - 1.0
    plan = S.Plan(n, pde, layout=S.LAYOUT_AOSOA, q_stride=m, out_stride=m)
    out = plan.alloc_output(E)
    dt = 0.5 / (3.0 * pde.max_wavespeed() * (2 * n - 1))
    for _ in range(warmup):
        plan.predict(q, dt, out=out)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(steps):
        plan.predict(q, dt, out=out)
    ev1.record(stream)
    torch.cuda.synchronize()
    plan.status()
    ms = ev0.elapsed_time(ev1) / steps
    del q, out
    return {"workload": f"dense LinearPde (m = {m}, every A_d / B_d entry nonzero), nDof {n}, {E} elements, "
                        "Q~U[-1,1] (user LinearPde path)",
            "elements_per_s": E / (ms * 1e-3), "ms_per_step": ms,
            "kernel": "stp_general_kernel" if os.environ.get("ADERSTP_NO_GDENSE") == "1" or n != 8 or m > 21
            else "stp_gdense_kernel"}


def measure_timestep(S, n, e, steps, warmup):
    """One full time step of the GPU solver on an e^3 periodic mesh: the
    predictor on the 1/h-scaled PDE without favg (the corrector never reads it, solver.cpp:184-253)
    followed by the corrector, per-element elastic material.  Device timing of each part."""
    import torch
    E = e ** 3
    q, par = S.generate(0, SEED, n, 0, E, layout=S.LAYOUT_AOSOA, q_stride=9)
    rho, cp, cs = par[:, 0], par[:, 1], par[:, 2]
    mu = rho * cs * cs
    lam = rho * cp * cp - 2.0 * mu
    s = float(e)  # 1 / h on the unit domain
    par_s = torch.stack([lam * s, mu * s, rho / s], 1).contiguous()
    pred = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, par_kind=S.PAR_LAMBDA_MU_RHO)
    corr = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, par_kind=S.PAR_RHO_CP_CS)
    out = pred.alloc_output(E, want_favg=False)
    dt = 0.35 / e / (3.0 * float(cp.max()) * (2 * n - 1))

    def p_step():
        pred.predict(q, dt, par=par_s, out=out, want_favg=False)

    def c_step():
        corr.correct(q, e, out, par=par)

    stream = torch.cuda.current_stream()
    res = {}
    for name, fn in (("predictor", p_step), ("corrector", c_step), ("step", lambda: (p_step(), c_step()))):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(steps):
            fn()
        ev1.record(stream)
        torch.cuda.synchronize()
        res[name] = ev0.elapsed_time(ev1) / steps
    # aderstp_run_simulation: fused predictor (it also applies the volume term) + surface-only
    # corrector, one call for all steps (its buffers are allocated once per call)
    sim = S.Plan(n, S.elastic_pde(), layout=S.LAYOUT_AOSOA, par_kind=S.PAR_RHO_CP_CS)
    sim.run_simulation(q, e, dt, par=par, cfl=0.35)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    ok, nsteps, _ = sim.run_simulation(q, e, steps * dt * (1 - 1e-12), par=par, cfl=0.35)
    ev1.record(stream)
    torch.cuda.synchronize()
    res["run_simulation_step"] = ev0.elapsed_time(ev1) / max(nsteps, 1)
    res["run_simulation_steps"] = nsteps
    res["run_simulation_stable"] = ok
    pred.status()
    m = 9
    corr_bytes = 8 * (3 * n ** 3 * m + 24 * n * n * m + 3)  # u in/out, qavg, own + neighbour faces, par
    peak = hbm_peak()[0] / 1e9
    return {"workload": f"GPU time step, elastic nDof {n}, periodic {e}^3 mesh ({E} elements), per-element material",
            "elements_per_s": E / (res["step"] * 1e-3), "ms_per_step": res["step"],
            "predictor_ms": res["predictor"], "corrector_ms": res["corrector"],
            "run_simulation_ms_per_step": res["run_simulation_step"],
            "run_simulation_steps": res["run_simulation_steps"], "run_simulation_stable": res["run_simulation_stable"],
            "run_simulation_elements_per_s": E / (res["run_simulation_step"] * 1e-3),
            "corrector_bytes_per_element": corr_bytes,
            "corrector_achieved_gbs": E * corr_bytes / (res["corrector"] * 1e-3) / 1e9,
            "corrector_hbm_frac": E * corr_bytes / (res["corrector"] * 1e-3) / 1e9 / peak,
            "bound": "predictor fp64, corrector hbm"}


def measure_e2e(S, plan, cfg, world, rank, dt, steps):
    """Same metric through the host-buffer public API (aderstp_predict_batch_host): pinned host
    inputs and outputs, host->device and device->host copies inside the timed region.  One GPU
    runs its full batch (<= 131,072 elements); with N > 1 ranks each rank uses <= 32,768 elements
    so that N pinned copies fit in the host's memory."""
    import torch
    n = cfg["n"]
    sh = shard_of(cfg, world, rank)
    E = min(sh.count, 131072 if world == 1 else 32768)
    grid = round(cfg["elems"] ** (1.0 / 3.0)) if cfg["dist"] == 2 else 1
    q_d, par_d = S.generate(cfg["dist"], SEED, n, sh.start, E, grid=grid, layout=S.LAYOUT_AOSOA,
                            q_stride=cfg["q_stride"])
    pin = lambda *shape: torch.empty(*shape, dtype=torch.float64, pin_memory=True)  # noqa: E731
    q_h = pin(E, plan.q_size)
    par_h = pin(E, 3)
    q_h.copy_(q_d)
    par_h.copy_(par_d)
    del q_d, par_d
    out_h = S.PredictorOutput(pin(E, plan.out_size).numpy(), pin(E, 3, plan.out_size).numpy(),
                              pin(E, 6, plan.face_size).numpy(), pin(E, 6, plan.face_size).numpy())
    qn, pn = q_h.numpy(), par_h.numpy()
    plan.predict_host(qn, dt, par=pn, out=out_h)  # warm-up (allocates the plan's chunk buffers)
    barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        plan.predict_host(qn, dt, par=pn, out=out_h)
    sec = max_over_ranks((time.perf_counter() - t0) / steps, device="cuda")
    barrier()
    h2d = E * (plan.q_size + 3) * 8
    d2h = E * (plan.out_size * 4 + plan.face_size * 12) * 8
    return dict(value=world * E / sec, unit=UNIT, h2d_bytes_per_step=h2d, d2h_bytes_per_step=d2h,
                ms_per_step=sec * 1e3, steps=steps, elements_per_rank=E,
                api="aderstp_predict_batch_host (pinned host buffers, copies pipelined on 3 streams)")


def host_cpu_info():
    """CPU model and the cores this process may run on (the reference's OpenMP threads are pinned
    one per core: OMP_PROC_BIND=close, OMP_PLACES=cores, set before libgomp initialises)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "cores_available": HOST_CORES, "os_cpu_count": os.cpu_count(),
            "pinning": "OMP_PROC_BIND=%s OMP_PLACES=%s" % (os.environ.get("OMP_PROC_BIND"),
                                                           os.environ.get("OMP_PLACES"))}


def repo_libraries_mapped():
    """Shared objects from this repository mapped into this process (/proc/self/maps): the
    reference arm must show only oracle/_ref, never paper_2003_12787_b200/libaderstp.so."""
    libs = set()
    try:
        with open("/proc/self/maps") as f:
            for ln in f:
                p = ln.split()[-1] if ln.strip() else ""
                if p.endswith(".so") and os.path.realpath(p).startswith(os.path.realpath(ROOT)):
                    libs.add(os.path.relpath(os.path.realpath(p), os.path.realpath(ROOT)))
    except OSError:
        pass
    return sorted(libs)


def _pin_openmp():
    # must run before oracle/_ref (and its libgomp) is loaded into this process
    os.environ.setdefault("OMP_PROC_BIND", "close")
    os.environ.setdefault("OMP_PLACES", "cores")


class CpuReference:
    """The reference's own CPU STP (oracle/_ref: the unmodified sources compiled by
    oracle/Makefile), driven like its production caller -- an OpenMP loop over elements, one
    ScratchArena per thread, predict(splitck | splitck_aosoa) + extrapolate_faces, one
    elastic_pde per element (proj/src/solver.cpp:334-345) -- on elements 0..sample-1 of the
    config's seeded workload with the config's dt.  Falls back to the C restatement (kind "port")
    only where oracle/_ref was not built."""

    def __init__(self, name, sample=None, threads=None):
        _pin_openmp()
        import oracle as O
        self.O, self.name, self.cfg = O, name, CONFIGS[name]
        n = self.cfg["n"]
        self.sample = sample or REFERENCE_SAMPLE[name]
        orc = O.Oracle()
        grid = round(self.cfg["elems"] ** (1.0 / 3.0)) if self.cfg["dist"] == 2 else 1
        self.q, par = orc.generate(self.cfg["dist"], SEED, n, 0, self.sample, grid=grid)
        self.lmr = orc.material_lmr(par)
        self.dt = config_dt(n)
        self.threads = threads or host_cpu_info()["cores_available"]
        self.ref = O.Reference() if O.reference_available() else None
        self.orc = orc
        self.kind = "reference" if self.ref else "port"
        self.variant = None

    def run_once(self, variant, threads=None, count=None):
        """Seconds of one predict loop over the sample (or its first `count` elements)."""
        n, t = self.cfg["n"], threads or self.threads
        q, lmr = (self.q, self.lmr) if count is None else (self.q[:count], self.lmr[:count])
        if self.ref is not None:
            return self.ref.stp(n, 9, q, self.dt, par=lmr, variant=variant, threads=t).seconds
        t0 = time.perf_counter()
        self.orc.stp(n, 9, q, self.dt, par=lmr, threads=t)
        return time.perf_counter() - t0

    def pick_variant(self):
        """The faster of splitck / splitck_aosoa on this host (one timed pass each)."""
        if self.ref is None:
            self.variant = "oracle/stp_oracle.c"
        elif self.variant is None:
            self.variant = min(("splitck", "aosoa"), key=lambda v: self.run_once(v))
        return self.variant

    def best_of(self, reps=REFERENCE_REPS):
        v = self.pick_variant()
        return min(self.run_once(v) for _ in range(reps))

    def describe(self, value, reps):
        lib = os.path.basename(self.ref.path) if self.ref else "oracle/libstp_oracle.so"
        info = host_cpu_info()
        return dict(value=value, unit=UNIT, cores=self.threads, kind=self.kind,
                    sample=f"elements 0..{self.sample - 1} of {self.cfg['desc'].split(':')[0]} "
                           f"({self.sample} of {self.cfg['elems']} elements; same seed, material and dt), "
                           f"best of {reps} reps, variant {self.variant} ({lib}), {self.threads} threads, "
                           "predict + extrapolate_faces loop",
                    cpu_model=info["cpu_model"], pinning=info["pinning"],
                    extrapolation="elements/s of the sample = elements/s of the full workload "
                                  "(elements are independent)")


def cpu_reference_run(name, reps=REFERENCE_REPS, single_core=False):
    """cpu_baseline of our arm: the same measurement as the reference arm, once, in a child
    process (our process has torch's OpenMP runtime loaded, so the reference's threads could not
    be pinned here)."""
    import subprocess
    env = dict(os.environ, OMP_PROC_BIND="close", OMP_PLACES="cores")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, os.path.abspath(__file__), "--impl", "reference", "--config", name, "--cpu-baseline-only"]
    if single_core:
        cmd.append("--single-core")
    r = subprocess.run(cmd, env=env, capture_output=True, text=True)
    if r.returncode != 0:
        return {"value": None, "unit": UNIT, "error": r.stderr.strip()[-500:]}
    return json.loads(r.stdout.strip().splitlines()[-1])


def _cpu_reference_measure(name, reps=REFERENCE_REPS, single_core=False):
    cr = CpuReference(name)
    best = cr.best_of(reps)
    out = cr.describe(cr.sample / best, reps)
    if single_core and cr.ref is not None and cr.threads > 1:  # also report 1 core
        one = max(64, cr.sample // cr.threads)
        r1 = min(cr.run_once(cr.variant, threads=1, count=one) for _ in range(reps))
        out["single_core_value"] = one / r1
        out["single_core_sample"] = f"{one} elements, 1 thread, variant {cr.variant}"
    return out


def run_reference_arm(args, world, rank):
    """--impl reference: rank 0 alone times the reference CPU STP on the same config; every
    timed step is the best of REFERENCE_REPS passes over the fixed sample."""
    if rank != 0:
        return 0
    cr = CpuReference(args.config)
    cr.pick_variant()
    values = []
    for i in range(args.warmup + args.steps):
        best = cr.best_of()
        if i >= args.warmup:
            values.append(cr.sample / best)
    value = statistics.median(values)
    info = cr.describe(value, REFERENCE_REPS)
    info["steps_values"] = values
    cfg = CONFIGS[args.config]
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": cr.sample / value * 1e3,
            "higher_is_better": True, "scaling": "strong" if cfg.get("strong") else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded SplitMix64, same generator, seed, material and dt as our arm)",
            "config": config_of(args.config, world),
            "reference_sample_elements": cr.sample,
            "repo_libraries_mapped": repo_libraries_mapped(),
            "cpu_baseline": info,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def roofline_of(S, n, per_gpu, elements_per_launch, traffic):
    flop_e, byte_e = S.flop_count(n, 9), S.byte_count(n, 9, True)
    fp64, fp64_src = fp64_peak()
    hbm, hbm_src = hbm_peak()
    tf = per_gpu * flop_e / 1e12
    gbs = per_gpu * byte_e / 1e9
    roof = min(fp64 / flop_e, hbm / byte_e)
    common = {"traffic": traffic, "flop_per_element": flop_e, "byte_per_element": byte_e,
              "roofline_elements_per_s": roof, "elements_per_launch": elements_per_launch}
    if fp64 / flop_e < hbm / byte_e:
        return dict({"bound": "fp64", "achieved": tf, "peak": fp64 / 1e12, "unit": "TFLOP/s",
                     "frac": tf / (fp64 / 1e12),
                     "peak_source": fp64_src,
                     "hbm_achieved_gbs": gbs, "hbm_frac": gbs / (hbm / 1e9)}, **common)
    return dict({"bound": "hbm", "achieved": gbs, "peak": hbm / 1e9, "unit": "GB/s", "frac": gbs / (hbm / 1e9),
                 "peak_source": hbm_src, "fp64_achieved_tflops": tf, "fp64_frac": tf / (fp64 / 1e12)}, **common)


def self_launch(args):
    """`bench.py --gpus N` outside torchrun: relaunch this command as N ranks (one process per
    GPU) under torch.distributed.run on 127.0.0.1, exactly as the driver does, and pass the
    rank-0 line through."""
    import socket
    import subprocess
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ, ADERSTP_BENCH_SELF_LAUNCHED="1", OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.run(cmd, env=env).returncode


def dry_run(args, world, rank):
    """--dry-run: the multi-rank flow without kernels (CPU, gloo): shards, the post-timing
    reductions and the rank-0 line.  Validates the launcher; never a measurement."""
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    cfg = CONFIGS[args.config]
    sh = shard_of(cfg, world, rank)
    starts = sum_over_ranks(float(sh.start))
    counts = sum_over_ranks(float(sh.count))
    c5 = {name: sum_over_ranks(float(shard_of(CONFIGS[name], world, rank).count)) for name in ("c5", "c5n6")}
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world, "dry_run": True,
                          "config": config_of(args.config, world), "shard_elements_total": counts,
                          "shard_starts_sum": starts, "c5_elements_total": c5}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def measure_scaling_leg(S, name, world, rank, steps, warmup):
    """BASELINE configs[4]: 1,048,576 elements split evenly over the GPUs (strong scaling);
    per-GPU and whole-box elements/s, device-resident, max over ranks."""
    c = CONFIGS[name]
    r = measure_device(S, c, world, rank, steps, warmup, want_clocks=False)
    whole = c["elems"] / (r["ms"] * 1e-3)
    rf = roofline_of(S, c["n"], whole / world, r["elements_per_launch"], None)
    return {"workload": c["desc"], "n_dof": c["n"], "global_elements": c["elems"], "n_gpus": world,
            "elements_per_gpu": r["shard"].count, "launches_per_gpu_step": r["launches_per_step"],
            "elements_per_launch": r["elements_per_launch"], "ms_per_step": r["ms"],
            "elements_per_s": whole, "elements_per_s_per_gpu": whole / world,
            "frac_of_roofline_per_gpu": rf["frac"], "bound": rf["bound"], "checksum": r["checksum"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c3")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true")
    ap.add_argument("--no-scaling", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="multi-rank plumbing only (CPU, gloo)")
    ap.add_argument("--cpu-baseline-only", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--single-core", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, _ = env_world()
    if args.impl == "reference" and args.cpu_baseline_only:
        print(json.dumps(_cpu_reference_measure(args.config, single_core=args.single_core)), flush=True)
        return 0
    if args.impl == "reference":
        # rank 0 alone times the host CPU; without torchrun there is nothing to launch
        return run_reference_arm(args, max(world, args.gpus), rank)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_launch(args)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dry_run:
        return dry_run(args, world, rank)

    import paper_2003_12787_b200 as S

    world, rank, _ = dist_setup()
    cfg = CONFIGS[args.config]
    n = cfg["n"]
    res = measure_device(S, cfg, world, rank, args.steps, args.warmup)
    ms = res["ms"]
    total = cfg["elems"] if cfg.get("strong") else world * cfg["elems"]
    value = total / (ms * 1e-3)
    per_gpu = value / world
    ncu_cfg = "c3" if args.config == "c5" else args.config
    roofline = roofline_of(S, n, per_gpu, res["elements_per_launch"], load_traffic(ncu_cfg, res["elements_per_launch"]))
    # physical pipe utilisation of the same kernel (ncu, profiles/ncu_summary.json): the elastic
    # kernels do ~2/3 of the algorithmic FLOPs (sparse flux), so this is the truth beside `frac`
    roofline["ncu_fp64_pipe_pct"] = load_ncu_field(ncu_cfg, "fp64_pipe_pct")
    roofline["ncu_dmma_pipe_pct"] = load_ncu_field(ncu_cfg, "dmma_pipe_pct")
    roofline["ncu_lsu_wavefront_pct"] = load_ncu_field(ncu_cfg, "lsu_wavefront_pct")

    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(S, res["plan"], cfg, world, rank, res["dt"], args.e2e_steps)

    # BASELINE configs[4] (C5) at every GPU count: nDof 8 and nDof 6, 1,048,576 elements split
    scaling = {}
    if not args.no_scaling:
        for name in ("c5", "c5n6"):
            if name != args.config:
                scaling[name] = measure_scaling_leg(S, name, world, rank, max(5, args.steps // 4), 3)

    others = {}
    if not args.no_other_configs and world == 1:
        for name in ("c1", "n4", "c2", "c4", "n9"):
            if name == args.config:
                continue
            c = CONFIGS[name]
            r = measure_device(S, c, 1, 0, max(5, args.steps // 4), 3, want_clocks=False)
            pg = c["elems"] / (r["ms"] * 1e-3)
            rf = roofline_of(S, c["n"], pg, c["elems"], load_traffic(name, c["elems"]))
            others[name] = {"workload": c["desc"], "elements_per_s": pg, "ms_per_step": r["ms"], "cuda_graph": r["cuda_graph"],
                            "fp64_gflops": pg * rf["flop_per_element"] / 1e9,
                            "achieved_gbs": pg * rf["byte_per_element"] / 1e9,
                            "roofline_elements_per_s": rf["roofline_elements_per_s"],
                            "frac_of_roofline": pg / rf["roofline_elements_per_s"], "bound": rf["bound"]}
        others["timestep_n8"] = measure_timestep(S, 8, 50, max(5, args.steps // 4), 3)
        others["c3_reference_layout"] = measure_reference_layout(S, CONFIGS["c3"], max(5, args.steps // 4), 3)
        others["table_pde_advection_m8_n8"] = measure_table_pde(S, max(5, args.steps // 4), 3)
        others["table_pde_advection_m8_n10"] = measure_table_pde(S, max(5, args.steps // 4), 3, n=10, E=16384)
        others["general_pde_dense_m21_n8"] = measure_general_pde(S, max(3, args.steps // 8), 3)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_reference_run(args.config, single_core=(world == 1))

    if rank == 0:
        E = res["shard"].count
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong" if cfg.get("strong") else "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded SplitMix64 stream, generated on device; per-element rho~U[2,3], "
                        "cp~U[4,6], cs~U[2,3.5])",
                "config": config_of(args.config, world),
                "run": {"elements_this_rank0": E, "launches_per_step": res["launches_per_step"],
                        "cuda_graph": res["cuda_graph"], "elements_per_launch": res["elements_per_launch"]},
                "fp64_gflops_per_gpu": per_gpu * roofline["flop_per_element"] / 1e9,
                "elements_per_s_per_gpu": per_gpu,
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": args.steps * res["launches_per_step"],
                "clocks": res["clocks"], "checksum": res["checksum"],
                "c5_strong_scaling": scaling, "other_configs": others}
        print(json.dumps(line), flush=True)
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

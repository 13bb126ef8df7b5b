# Multi-rank flow of bench.py on a 1-GPU box: 2 ranks sharing cuda:0 over gloo (plumbing check
# only -- the numbers of such a run are not measurements).  The reference arm under torchrun too.
exec > gpurun_out/multirank.log 2>&1
export ADERSTP_BENCH_BACKEND=gloo
for cfg in c3 c5; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --steps 3 --warmup 3 --config $cfg --e2e-steps 1; echo "rc=$? ($cfg)"
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 2 --steps 1 --warmup 1 --impl reference; echo "rc=$? (reference arm)"

# full GPU test suite, smoke, default bench, reference arm (round-end style)
exec > gpurun_out/final.log 2>&1
python -m pytest tests -m gpu -q 2>&1 | tail -5
python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_final_ref.json 2>> gpurun_out/bench_final.err; echo "ref rc=$?"

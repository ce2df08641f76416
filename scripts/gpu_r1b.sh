set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25
for c in 2 3 5; do
  timeout -s KILL 300 python bench.py --config $c --steps 50 --warmup 5 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; tail -3 gpurun_out/bench_c$c.err
  cat gpurun_out/bench_c$c.json
done

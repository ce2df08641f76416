for dbg in 0 1 6 3 5; do
  CO_TC_DEBUG=$dbg timeout -s KILL 300 python bench.py --config 2 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; tail -1 gpurun_out/d.err
  python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C2 dbg=$dbg', j['roofline']['ms_per_launch'])"
done
for dbg in 0 1 6; do
  CO_TC_DEBUG=$dbg timeout -s KILL 300 python bench.py --config 5 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; tail -1 gpurun_out/d.err
  python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C5 dbg=$dbg', j['roofline']['ms_per_launch'])"
done

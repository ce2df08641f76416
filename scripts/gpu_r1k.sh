python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for dbg in 0 1 2 4 3 6 5; do
  for eg in 2 3; do
  CO_TC_EG=$eg CO_TC_DEBUG=$dbg timeout -s KILL 300 python bench.py --config 2 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; tail -2 gpurun_out/d.err
  python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C2 dbg=$dbg eg=$eg', j['roofline']['kernel'], j['roofline']['ms_per_launch'])"
  done
done
for dbg in 0 1 2; do
  CO_TC_DEBUG=$dbg timeout -s KILL 300 python bench.py --config 5 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; tail -2 gpurun_out/d.err
  python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C5 dbg=$dbg', j['roofline']['kernel'], j['roofline']['ms_per_launch'])"
  CO_TC_DEBUG=$dbg timeout -s KILL 300 python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; tail -2 gpurun_out/d.err
  python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C4 dbg=$dbg', [(l['kernel'], l['ms_per_launch']) for l in j['layers']])"
done

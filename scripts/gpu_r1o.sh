timeout -s KILL 600 python -m pytest tests/test_gpu_dense_tc.py -x -q 2>&1 | tail -2
for eg in 2 3; do
  CO_TC_EG=$eg timeout -s KILL 300 python bench.py --config 2 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; tail -2 gpurun_out/d.err
  python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C2 eg=$eg', j['roofline']['kernel'], j['roofline']['ms_per_launch'], j['roofline']['frac'])"
done
CO_TC_DEBUG=6 timeout -s KILL 300 python bench.py --config 2 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C2 dbg6', j['roofline']['kernel'], j['roofline']['ms_per_launch'])"
timeout -s KILL 300 python bench.py --config 5 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C5', j['roofline']['kernel'], j['roofline']['ms_per_launch'], j['roofline']['frac'])"
timeout -s KILL 300 python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C4', j['value'], [(l['kernel'], l['ms_per_launch'], l['frac']) for l in j['layers']])"

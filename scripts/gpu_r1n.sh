timeout -s KILL 600 python -m pytest tests/test_gpu_dense_tc.py -x -q 2>&1 | tail -2
for v in "" nohint; do for eg in 2 3; do
  CO_LIB_VARIANT=$v CO_TC_EG=$eg timeout -s KILL 300 python bench.py --config 2 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; tail -2 gpurun_out/d.err
  python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C2 v=$v eg=$eg', j['roofline']['kernel'], j['roofline']['ms_per_launch'], j['roofline']['frac'])"
done; done
for v in "" nohint; do CO_LIB_VARIANT=$v CO_TC_DEBUG=6 timeout -s KILL 300 python bench.py --config 2 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C2 dbg6 v=$v', j['roofline']['kernel'], j['roofline']['ms_per_launch'])"; done
for v in "" nohint; do CO_LIB_VARIANT=$v timeout -s KILL 300 python bench.py --config 5 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C5 v=$v', j['roofline']['kernel'], j['roofline']['ms_per_launch'], j['roofline']['frac'])"; done

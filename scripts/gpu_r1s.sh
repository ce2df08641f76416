CO_TC_CS=2 timeout -s KILL 600 python -m pytest tests/test_gpu_dense_tc.py -x -q -k "halo_c2like" 2>&1 | tail -1
for cs in 1 2; do for eg in 2 3; do
  CO_TC_CS=$cs CO_TC_EG=$eg timeout -s KILL 300 python bench.py --config 2 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; tail -1 gpurun_out/d.err
  python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C2 cs=$cs eg=$eg', j['roofline']['kernel'], j['roofline']['ms_per_launch'], j['roofline']['frac'])"
done; done

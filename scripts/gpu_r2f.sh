CO_TC_SWA=1 timeout -s KILL 300 python -m pytest tests/test_gpu_dense_tc.py -x -q -k "halo_c2like or halo_kt1 or cta_pair" 2>&1 | tail -3
for pair in 1 2; do for swa in 0 1; do for dbg in 0 3; do
  CO_TC_SWA=$swa CO_TC_PAIR=$pair CO_TC_EG=3 CO_TC_DEBUG=$dbg timeout -s KILL 300 python bench.py --config 2 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; tail -1 gpurun_out/d.err
  python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C2 pair=$pair swa=$swa dbg=$dbg', j['roofline']['ms_per_launch'], j['roofline']['frac'])"
done; done; done

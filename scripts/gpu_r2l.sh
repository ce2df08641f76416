timeout -s KILL 300 python -m pytest tests/test_gpu_dense_tc.py -x -q -k "halo_c2like" 2>&1 | tail -1
for dbg in 0 1 5 3; do
  CO_LOG=1 CO_TC_DEBUG=$dbg timeout -s KILL 300 python bench.py --config 2 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; grep "\[co\]" gpurun_out/d.err | head -1
  python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C2 dbg=$dbg', j['roofline']['kernel'], j['roofline']['ms_per_launch'], j['roofline']['frac'])"
done
CO_TC_PAIR=1 timeout -s KILL 300 python bench.py --config 2 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C2 single', j['roofline']['kernel'], j['roofline']['ms_per_launch'], j['roofline']['frac'])"

python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
CO_TC_PIPE=1 timeout -s KILL 900 python -m pytest tests/test_gpu_dense_tc.py -x -q -k "halo_c2like" 2>&1 | tail -2
for pipe in 0 1; do for dbg in 0 4; do
  CO_TC_PIPE=$pipe CO_TC_DEBUG=$dbg timeout -s KILL 300 python bench.py --config 2 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; tail -2 gpurun_out/d.err
  python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C2 pipe=$pipe dbg=$dbg', j['roofline']['kernel'], j['roofline']['ms_per_launch'], j['roofline']['frac'])"
done; done
B3="python bench.py --config 3 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
$B3 > gpurun_out/p3.log 2>&1 && timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_step_dw -s 40 -c 2 -o gpurun_out/prof_c3s $B3 > gpurun_out/ncu_c3.log 2>&1
tail -1 gpurun_out/ncu_c3.log

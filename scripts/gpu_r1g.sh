python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout -s KILL 900 python -m pytest tests/test_gpu_dense_tc.py -x -q 2>&1 | tail -3
for eg in 2 3 4; do
  CO_TC_EG=$eg timeout -s KILL 300 python bench.py --config 2 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/c2_eg$eg.json 2> gpurun_out/c2_eg$eg.err; tail -2 gpurun_out/c2_eg$eg.err
  python -c "import json;j=json.load(open('gpurun_out/c2_eg$eg.json'));print('EG$eg', j['value'], j['roofline']['kernel'], j['roofline']['frac'], j['roofline']['ms_per_launch'])"
done
timeout -s KILL 300 python bench.py --config 5 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/c5.json 2> gpurun_out/c5.err; tail -2 gpurun_out/c5.err
python -c "import json;j=json.load(open('gpurun_out/c5.json'));print('C5', j['value'], j['roofline']['kernel'], j['roofline']['frac'], j['roofline']['ms_per_launch'])"
B="python bench.py --config 2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
CO_TC_EG=3 $B > gpurun_out/plain_c2.log 2>&1 && CO_TC_EG=3 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_step_dense_tc -s 3 -c 1 -o gpurun_out/prof_c2_v5 $B > gpurun_out/ncu_c2.log 2>&1
tail -1 gpurun_out/ncu_c2.log

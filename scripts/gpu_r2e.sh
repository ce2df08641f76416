for dbg in 0 1 6 3 5; do
  CO_TC_PAIR=2 CO_TC_EG=3 CO_TC_DEBUG=$dbg timeout -s KILL 300 python bench.py --config 2 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; tail -1 gpurun_out/d.err
  python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C2 pair dbg=$dbg', j['roofline']['ms_per_launch'])"
done
B="python bench.py --config 2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
CO_TC_PAIR=2 CO_TC_EG=3 $B > gpurun_out/p.log 2>&1 && CO_TC_PAIR=2 CO_TC_EG=3 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_step_dense_tc -s 5 -c 1 -o gpurun_out/prof_c2_pair $B > gpurun_out/ncu.log 2>&1; tail -1 gpurun_out/ncu.log

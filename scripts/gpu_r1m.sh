B="python bench.py --config 2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
CO_TC_DEBUG=6 $B > gpurun_out/p.log 2>&1 && CO_TC_DEBUG=6 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_step_dense_tc -s 5 -c 1 -o gpurun_out/prof_c2_dbg6 $B > gpurun_out/ncu.log 2>&1
tail -1 gpurun_out/ncu.log

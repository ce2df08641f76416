scripts/bw_probe 0 256 1 1 > gpurun_out/probe.log 2>&1 && ncu --set full --clock-control none -c 1 -s 2 -o gpurun_out/prof_probe scripts/bw_probe 0 256 1 1 > gpurun_out/ncu_probe.log 2>&1
B="python bench.py --config 2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
CO_TC_DEBUG=6 $B > gpurun_out/p.log 2>&1 && CO_TC_DEBUG=6 ncu --set full --clock-control none -k regex:k_step_dense_tc -s 5 -c 1 -o gpurun_out/prof_d6b $B > gpurun_out/ncu_d6.log 2>&1
tail -1 gpurun_out/ncu_probe.log gpurun_out/ncu_d6.log

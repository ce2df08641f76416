python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -2 gpurun_out/bench_default.err; cat gpurun_out/bench_default.json
for c in 1 3 4 5; do timeout -s KILL 600 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; tail -1 gpurun_out/bench_c$c.err; done
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain_default.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv $B > gpurun_out/ncu_l.log 2>&1
B2="python bench.py --config 2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
$B2 > gpurun_out/p2.log 2>&1 && timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_step_dense -s 5 -c 1 -o gpurun_out/prof2_c2 $B2 > gpurun_out/ncu_c2.log 2>&1
B3="python bench.py --config 3 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
$B3 > gpurun_out/p3.log 2>&1 && timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_step_dw -s 40 -c 2 -o gpurun_out/prof2_c3 $B3 > gpurun_out/ncu_c3.log 2>&1
B5="python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
$B5 > gpurun_out/p5.log 2>&1 && timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_step_dense -s 20 -c 1 -o gpurun_out/prof2_c5 $B5 > gpurun_out/ncu_c5.log 2>&1
B4="python bench.py --config 4 --steps 30 --warmup 3 --no-e2e --no-cpu-baseline"
$B4 > gpurun_out/p4.log 2>&1 && timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_step_dense -s 100 -c 5 -o gpurun_out/prof2_c4 $B4 > gpurun_out/ncu_c4.log 2>&1
ls gpurun_out/*.ncu-rep

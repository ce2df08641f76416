set -x
timeout -s KILL 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout -s KILL 300 python bench.py > gpurun_out/bench_r1a.json 2> gpurun_out/bench_r1a.err; tail -3 gpurun_out/bench_r1a.err
cat gpurun_out/bench_r1a.json
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1a.csv $B > gpurun_out/ncu1.log 2>&1
$B > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_step_dense_tc -s 5 -c 1 -o gpurun_out/prof_dense_r1a $B > gpurun_out/ncu2.log 2>&1
ls -la gpurun_out

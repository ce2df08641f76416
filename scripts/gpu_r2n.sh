timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
CO_LOG=1 timeout -s KILL 400 python bench.py --config 4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c4.json 2> gpurun_out/c4.err; grep "\[co\]" gpurun_out/c4.err | sort -u; python -c "import json;j=json.load(open('gpurun_out/c4.json'));print('C4', j['value'], [(l['kernel'], l['ms_per_launch'], l['frac']) for l in (j['layers'] or [])])"
B4="python bench.py --config 4 --steps 30 --warmup 3 --no-e2e --no-cpu-baseline"
$B4 > gpurun_out/p4.log 2>&1 && timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_step_dense -s 100 -c 5 -o gpurun_out/prof3_c4 $B4 > gpurun_out/ncu_c4.log 2>&1; tail -1 gpurun_out/ncu_c4.log

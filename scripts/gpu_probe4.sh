P=scripts/bw_probe
for m in 0 3 4; do $P $m 256 1 1; $P $m 384 1 1; done
for dbg in 6 0; do CO_TC_DEBUG=$dbg timeout -s KILL 120 python bench.py --config 2 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C2 dbg$dbg', j['roofline']['ms_per_launch'])"; done

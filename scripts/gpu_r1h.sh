python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
CO_LOG=1 timeout -s KILL 900 python -m pytest tests/test_gpu_dense_tc.py -x -q 2>&1 | tail -25
timeout -s KILL 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
CO_LOG=1 timeout -s KILL 600 python bench.py --config 4 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c4.json 2> gpurun_out/c4.err; tail -8 gpurun_out/c4.err
python -c "import json;j=json.load(open('gpurun_out/c4.json'));print('C4', j['value'], j['ms_per_step'], [(l['kernel'], l['bound'], l['frac'], l['ms_per_launch']) for l in j['layers']])"
for c in 2 3 5; do timeout -s KILL 300 python bench.py --config $c --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/c$c.json 2> gpurun_out/c$c.err; tail -2 gpurun_out/c$c.err; python -c "import json;j=json.load(open('gpurun_out/c$c.json'));print('C$c', j['value'], j['roofline']['kernel'], j['roofline']['frac'], j['roofline']['ms_per_launch'])"; done

timeout -s KILL 600 python -m pytest tests/test_gpu_depthwise.py -x -q 2>&1 | tail -2
for v in "" px2 px3; do
CO_LIB_VARIANT=$v timeout -s KILL 300 python bench.py --config 3 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; tail -1 gpurun_out/d.err; python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C3 v=$v', j['value'], [(l['kernel'], l['ms_per_launch'], l['frac']) for l in j['layers']])"
done
CO_LIB_VARIANT=px2 timeout -s KILL 600 python -m pytest tests/test_gpu_depthwise.py -x -q 2>&1 | tail -1

for v in "" nb2m3 nb2m4 nb4m2 nb3m3 st3; do
CO_LIB_VARIANT=$v timeout -s KILL 300 python bench.py --config 3 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; tail -1 gpurun_out/d.err; python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C3 v=$v', j['value'], [(l['kernel'], l['ms_per_launch'], l['frac']) for l in j['layers']])"
done

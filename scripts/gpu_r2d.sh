for pair in 1 2; do for eg in 2 3; do
  CO_LOG=1 CO_TC_PAIR=$pair CO_TC_EG=$eg timeout -s KILL 300 python bench.py --config 2 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; grep "\[co\]" gpurun_out/d.err | head -1
  python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C2 pair=$pair eg=$eg', j['value'], j['roofline']['kernel'], j['roofline']['ms_per_launch'], j['roofline']['frac'])"
done; done
for pair in 1 2; do
  CO_LOG=1 CO_TC_PAIR=$pair timeout -s KILL 300 python bench.py --config 5 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; grep "\[co\]" gpurun_out/d.err | head -1
  python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C5 pair=$pair', j['value'], j['roofline']['kernel'], j['roofline']['ms_per_launch'], j['roofline']['frac'])"
done

for v in "CO_TC_EG=2" "CO_TC_EG=3" "CO_TC_CS=2 CO_TC_EG=2" "CO_TC_CS=2 CO_TC_EG=3"; do
  env $v timeout -s KILL 300 python bench.py --config 2 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/d.json 2> gpurun_out/d.err; tail -1 gpurun_out/d.err
  python -c "import json;j=json.load(open('gpurun_out/d.json'));print('C2 $v', j['roofline']['kernel'], j['roofline']['ms_per_launch'], j['roofline']['frac'])"
done

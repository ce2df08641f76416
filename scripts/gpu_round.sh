#!/usr/bin/env bash
# Round-end measurement flow on one B200 (run through gpurun from the repo root):
#   gpurun --timeout 3000 -- 'bash scripts/gpu_round.sh r1d'
# 1. build + the GPU test suite; 2. bench.py on every config (JSON lines under
# gpurun_out/bench_<tag>_c<N>.json) and the reference arm; 3. the companion
# benches (pooling, chunked steps, MHA); 4. the ncu launch list of the default
# bench command (after the same command exited 0 without ncu).  One ncu run per
# gpurun call: the `--set full` captures go through scripts/gpu_ncu_full.sh in
# calls of their own.  Summarise with scripts/ncu_summary.py and copy what is
# judged into profiles/.
set -u
TAG=${1:-rX}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout -s KILL 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
for c in 1 2 3 4 5; do
  timeout -s KILL 600 python bench.py --config $c --steps 100 --warmup 10 > $OUT/bench_${TAG}_c$c.json 2> $OUT/bench_${TAG}_c$c.err
  tail -c 300 $OUT/bench_${TAG}_c$c.json; echo
done
timeout -s KILL 600 python bench.py > $OUT/bench_${TAG}_default.json 2> $OUT/bench_${TAG}_default.err
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_${TAG}_ref.json 2> $OUT/bench_${TAG}_ref.err
timeout -s KILL 600 python scripts/bench_pool.py > $OUT/bench_${TAG}_pool.jsonl 2>&1
timeout -s KILL 600 python scripts/bench_chunked.py > $OUT/bench_${TAG}_chunked.jsonl 2>&1
timeout -s KILL 600 python scripts/bench_mha.py > $OUT/bench_${TAG}_mha.jsonl 2>&1
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
$B > $OUT/plain_${TAG}.log 2>&1 && \
  timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_${TAG}_c2.csv $B > $OUT/ncu_launches_${TAG}.log 2>&1
ls $OUT | tail -30

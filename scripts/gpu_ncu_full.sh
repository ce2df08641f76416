#!/usr/bin/env bash
# One `ncu --set full` capture per gpurun call, after the same command ran clean:
#   gpurun --timeout 1200 -- 'bash scripts/gpu_ncu_full.sh <tag> <kernel regex> <skip> <command...>'
# e.g.  bash scripts/gpu_ncu_full.sh r1d_c2 k_step_dense_tc 5 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e
set -u
TAG=$1; KREGEX=$2; SKIP=$3; shift 3
mkdir -p gpurun_out
"$@" > gpurun_out/plain_${TAG}.log 2>&1 || { echo "command failed without ncu"; exit 1; }
timeout -s KILL 900 ncu --set full --clock-control none --import-source on --kernel-name-base ${NCU_NAME_BASE:-function} -k "regex:$KREGEX" -s $SKIP -c 1 \
  -o gpurun_out/prof_${TAG} "$@" > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_full_${TAG}.log

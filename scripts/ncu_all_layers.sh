#!/bin/bash
# ncu --set full capture of every bench layer at a Ready step (GPU box; one
# layer per process via scripts/layer_probe.py, each run first without ncu).
# Usage: [KEEP="c4l2 c2l0"] bash scripts/ncu_all_layers.sh <tag>
#        -> gpurun_out/<tag>_c<C>l<L>[_raw].raw.csv (+ .ncu-rep for the KEEP list)
# Summarise here with scripts/ncu_summary.py (profiles/<tag>_*.txt, ncu_traffic.json).
set -u
TAG=${1:-r2}
mkdir -p gpurun_out
# config layer state kernel-regex launches-before-the-2nd-Ready-step
CASES="1 0 psum k_step_direct 3
2 0 psum k_step_dense_tc 3
3 0 psum k_step_dw 3
3 1 psum k_step_dw 5
4 0 psum k_step_dense_tc 5
4 1 psum k_step_dense_tc 1
4 2 psum k_step_dense_tc 3
4 3 psum k_step_dense_tc 3
4 4 psum k_step_dense_tc 3
5 0 psum k_step_dense_tc 17
5 0 raw k_step_dense_tc 1
4 0 raw k_step_stem_raw 1"
echo "$CASES" | while read C L S K N; do
  suf=""; [ "$S" = raw ] && suf="_raw"
  out=gpurun_out/${TAG}_c${C}l${L}${suf}
  st=$S; [ "$K" = k_step_stem_raw ] && st=auto           # the planner's RAW stem (other layers PSUM)
  python scripts/layer_probe.py --config $C --layer $L --state $st --steps 3 > $out.plain.log 2>&1 || { echo "plain run failed: $C $L $S"; continue; }
  ncu --set full --clock-control none --import-source on -k regex:$K -s $N -c 1 -o $out \
      python scripts/layer_probe.py --config $C --layer $L --state $st --steps 3 > $out.ncu.log 2>&1
  rc=$?
  # the raw metrics page travels back (the full reports would pass gpurun's 64 MiB limit);
  # reports named in KEEP stay whole for source-level reading
  ncu -i $out.ncu-rep --page raw --csv > $out.raw.csv 2>/dev/null
  case " ${KEEP:-} " in *" c${C}l${L}${suf} "*) ;; *) rm -f $out.ncu-rep ;; esac
  echo "$C $L $S rc=$rc $(tail -1 $out.plain.log)"
done

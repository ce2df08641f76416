P=scripts/bw_probe
for f in 0 1 2 3; do for sm in 0 204800; do $P 4 384 1 1 $((f*65536)) $sm; done; done

P=scripts/bw_probe
for t in 256 384; do $P 0 $t 1 1; $P 3 $t 1 1; done

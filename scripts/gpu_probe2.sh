P=scripts/bw_probe
for w in 0 100 250 500 1000 2000; do $P 0 256 1 1 $w; $P 0 384 1 1 $w; done

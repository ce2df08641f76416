P=scripts/bw_probe
for ni in 1 2 4; do $P 2 256 4 $ni; $P 2 512 2 $ni; done
for ni in 1 2 4; do $P 1 256 2 $ni; $P 1 256 4 $ni; $P 1 512 2 $ni; done
for ni in 1 2; do for t in 256 384 512; do $P 0 $t 1 $ni; done; $P 0 256 2 $ni; $P 0 256 3 $ni; $P 0 512 2 $ni; done

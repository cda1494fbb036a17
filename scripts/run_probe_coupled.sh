# lead experiment with the coupled probe (probe_tma_coupled.cu): F consumers 2 rows ahead (the
# phase kernels today) or 3 (needs a 4th z-ring slot: ~37 KB less for the stage rings)
P="timeout 20 scripts/probe_tma_coupled"
for d in 300 500; do
  $P 7 6 5 112 $d $d 3 2
  $P 7 6 5 112 $d $d 3 3
  $P 7 4 3 150 $d $d 3 3
  $P 7 4 3 150 $d $d 3 2
done
$P 7 6 5 112 500 100 3 3
$P 7 4 3 150 500 100 3 3

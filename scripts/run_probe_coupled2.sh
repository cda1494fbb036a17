P="timeout 30 scripts/probe_tma_coupled2"
for d in 0 300 500; do
  $P 128 7 6 5 112 $d $d
  $P 64 7 6 5 57 $d $d
  $P 64 7 5 5 57 $d $d
done
$P 128 7 6 5 112 500 100
$P 64 7 6 5 57 500 100
$P 128 7 6 5 112 100 500
$P 64 7 6 5 57 100 500

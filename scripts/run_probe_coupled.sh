# coupling experiment with the coupled probe (see probe_tma_coupled.cu): couple 0 none, 2 stage (sread), 3 stage + row (zready)
# (couple 1 alone lets F run rows ahead and alias the zready phases: not a valid configuration)
P="timeout 20 scripts/probe_tma_coupled"
for d in 0 300 500; do
  for c in 0 2 3; do $P 7 6 5 112 $d $d $c; done
done
$P 7 6 5 112 500 100 3
$P 7 6 5 112 100 500 3

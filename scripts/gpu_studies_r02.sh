# refresh the NEXT-1..4 studies with the round-2 code (profiles/r02_next*)
mkdir -p gpurun_out
timeout 600 python scripts/studies.py table1 --config C5 > gpurun_out/r02_next3_t1_c5.json 2> gpurun_out/t1.err; echo t1 rc $?
timeout 900 python scripts/studies.py table1 --config C4 --hard > gpurun_out/r02_next3_t1_hard.json 2> gpurun_out/t1h.err; echo t1h rc $?
timeout 600 python scripts/studies.py timestep --config C5 > gpurun_out/r02_next4_timestep.json 2> gpurun_out/ts.err; echo ts rc $?
timeout 900 python scripts/studies.py trisor --config C5 > gpurun_out/r02_next1_trisor.json 2> gpurun_out/tr.err; echo tr rc $?
timeout 900 python scripts/studies.py precision > gpurun_out/r02_next2_precision.json 2> gpurun_out/pr.err; echo pr rc $?
tail -2 gpurun_out/*.err

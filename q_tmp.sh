python bench.py --workload c3 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"boids_tile|boids_step" -s 3 -c 1 -o gpurun_out/prof_boids python bench.py --workload c3 > gpurun_out/ncu4.log 2>&1
python bench.py --workload c5 > gpurun_out/plain5.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"sir_sweep" -c 1 -o gpurun_out/prof_sweep python bench.py --workload c5 > gpurun_out/ncu5.log 2>&1
tail -1 gpurun_out/ncu4.log gpurun_out/ncu5.log

timeout 600 python -m pytest tests/test_gpu_walk.py tests/test_capi.py -x -q 2>&1 | tail -3
python bench.py --workload walk 2>&1 | tail -1
python bench.py --workload walk_scale 2>&1 | tail -1

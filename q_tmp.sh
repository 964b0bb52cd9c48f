timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python tools/measure_all.py > gpurun_out/all_configs.jsonl 2> gpurun_out/all_configs.err; cat gpurun_out/all_configs.jsonl | cut -c1-300

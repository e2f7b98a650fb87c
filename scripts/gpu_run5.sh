python -m pytest tests/test_gpu_top1.py -x -q --durations=5 > gpurun_out/top1.log 2>&1; tail -40 gpurun_out/top1.log

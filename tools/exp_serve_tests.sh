# serving GPU tests (live macro, FuDG, preemption, TP=2 pair macro, live mitosis) + TP tests on 2 GPUs
mkdir -p gpurun_out
timeout 1500 python -m pytest -q tests/test_gpu_serve.py tests/test_gpu_tp.py tests/test_gpu_migrate.py 2>&1 | tail -6 > gpurun_out/serve_tests.txt
cat gpurun_out/serve_tests.txt

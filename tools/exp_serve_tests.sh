# live mitosis GPU test x3 on 2 GPUs and once on one GPU
mkdir -p gpurun_out
: > gpurun_out/serve_tests.txt
for i in 1 2 3; do timeout 300 python -m pytest -q tests/test_gpu_serve.py -k mitosis 2>&1 | tail -12 >> gpurun_out/serve_tests.txt; done
CUDA_VISIBLE_DEVICES=0 timeout 300 python -m pytest -q tests/test_gpu_serve.py -k mitosis 2>&1 | tail -12 >> gpurun_out/serve_tests.txt
cat gpurun_out/serve_tests.txt

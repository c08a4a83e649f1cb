# 8B PaDG goodput at HEAD: macro of 4 instances (4 GPUs) and of 1 (1 GPU), ShareGPT 5 s / 100 ms, P90
mkdir -p gpurun_out
timeout 2400 python goodput_bench.py --gpus 4 --shape 8b --lo 40 --hi 800 --iters 6 --n-req 400 --duration 30 \
  > gpurun_out/goodput_8b_4gpu.jsonl 2> gpurun_out/goodput_8b_4gpu.err
timeout 1800 python goodput_bench.py --gpus 1 --shape 8b --lo 10 --hi 200 --iters 6 --n-req 400 --duration 30 \
  > gpurun_out/goodput_8b_1gpu.jsonl 2> gpurun_out/goodput_8b_1gpu.err
tail -1 gpurun_out/goodput_8b_4gpu.jsonl | cut -c1-300; tail -1 gpurun_out/goodput_8b_1gpu.jsonl | cut -c1-300

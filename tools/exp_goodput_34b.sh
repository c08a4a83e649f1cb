# configs[2]: 34B-shape macro of 4 single-GPU instances, ShareGPT 5 s / 100 ms, P90, at HEAD
mkdir -p gpurun_out
timeout 2400 python goodput_bench.py --gpus 4 --shape 34b --blocks 3000 --lo 8 --hi 256 --iters 6 --n-req 200 \
  --duration 30 > gpurun_out/goodput_34b_4gpu.jsonl 2> gpurun_out/goodput_34b_4gpu.err
tail -1 gpurun_out/goodput_34b_4gpu.jsonl | cut -c1-300

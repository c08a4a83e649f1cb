# configs[3]-like goodput: macro of TP=2 pairs of the 70B shape, 2 pairs (4 GPUs) and 1 pair (2 GPUs)
mkdir -p gpurun_out
timeout 2400 python goodput_bench.py --gpus 4 --tp 2 --shape 70b --blocks 4000 --lo 4 --hi 96 --iters 6 --n-req 200 \
  --duration 30 > gpurun_out/goodput_70b_tp2_4gpu.jsonl 2> gpurun_out/goodput_70b_tp2_4gpu.err
timeout 2400 python goodput_bench.py --gpus 2 --tp 2 --shape 70b --blocks 4000 --lo 4 --hi 96 --iters 6 --n-req 200 \
  --duration 30 > gpurun_out/goodput_70b_tp2_2gpu.jsonl 2> gpurun_out/goodput_70b_tp2_2gpu.err
tail -1 gpurun_out/goodput_70b_tp2_4gpu.jsonl | cut -c1-400; tail -1 gpurun_out/goodput_70b_tp2_2gpu.jsonl | cut -c1-400

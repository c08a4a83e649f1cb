# configs[4]: mitosis live on 4 B200s, 34B shape, long prompts, rate stepped 2 -> 5 -> 2 req/s
mkdir -p gpurun_out
timeout 3000 python tools/mitosis_live.py --gpus 4 --shape 34b --rates 2,7,2 --step-s 40 --window-s 20 --blocks 3000 \
  > gpurun_out/mitosis_live.jsonl 2> gpurun_out/mitosis_live.err
cat gpurun_out/mitosis_live.jsonl; tail -3 gpurun_out/mitosis_live.err

# configs[4]: mitosis with the automatic triggers on 4 B200s (34B, long prompts, 2 -> 7 -> 2 req/s)
mkdir -p gpurun_out
timeout 3000 python tools/mitosis_live.py --gpus 4 --shape 34b --rates 2,7,2 --step-s 40 --window-s 20 --blocks 3000 \
  --only mitosis-auto,mitosis > gpurun_out/mitosis_auto.jsonl 2> gpurun_out/mitosis_auto.err
cat gpurun_out/mitosis_auto.jsonl; tail -3 gpurun_out/mitosis_auto.err

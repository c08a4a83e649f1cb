# macro instance of TP=2 pairs (configs[3]): live-serving parity test + a 70B fixed-rate probe on 2 GPUs
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_serve.py -k "tp2" 2>&1 | tail -5 > gpurun_out/tp_serve_test.txt
timeout 1500 python goodput_bench.py --gpus 2 --tp 2 --shape 70b --blocks 4000 --rates 4,8 --n-req 120 --duration 30 \
  > gpurun_out/tp_serve_probe.jsonl 2> gpurun_out/tp_serve_probe.err
cat gpurun_out/tp_serve_test.txt gpurun_out/tp_serve_probe.jsonl; tail -5 gpurun_out/tp_serve_probe.err

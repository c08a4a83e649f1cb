mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_ops.py -k "attention_prefill" 2>&1 | tail -3 > gpurun_out/t128_ops.txt
o=gpurun_out/exp_t128.jsonl; : > $o
for i in 1 2; do
  for v in "ECOSERVE_ATTN_T128=0" "ECOSERVE_XX=1"; do
    env $v timeout 600 python tools/prefill_long_ab.py 8b 2 >> $o 2>> gpurun_out/exp_t128.err
    env $v timeout 600 python tools/prefill_long_ab.py 34b 2 >> $o 2>> gpurun_out/exp_t128.err
  done
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_t128.json 2> gpurun_out/bench_t128.err
cat gpurun_out/t128_ops.txt $o gpurun_out/bench_t128.json

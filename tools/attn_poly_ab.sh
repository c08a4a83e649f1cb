# prefill attention: default vs the opt-in 128-key kernel (attn_bench, L=32 pool) + parity
for v in "" "ECOSERVE_ATTN_T128=1" "ECOSERVE_ATTN_T128=2" ""; do
  echo "== $v"; env $v timeout 120 ./tools/attn_bench 32
done
echo "== tests"; timeout 900 python -m pytest -q -x tests/test_gpu_ops.py -k "prefill" 2>&1 | tail -3
timeout 1500 python -m pytest -q -x tests/test_gpu_fullsize.py -k "T128" 2>&1 | tail -3

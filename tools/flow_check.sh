timeout 600 python -m pytest -q -x tests/test_gpu_ops.py -k "stream_k" 2>&1 | tail -2
for i in 1 2 3; do
timeout 300 python tools/decode_ablate.py --one
ECOSERVE_ATTN_SK=0 timeout 300 python tools/decode_ablate.py --one
done

timeout 600 python -m pytest -q -x tests/test_gpu_ops.py -k "attention_decode" 2>&1 | tail -2
for i in 1 2; do
timeout 300 python tools/decode_ablate.py --one
ECOSERVE_ABLATE=1 timeout 300 python tools/decode_ablate.py --one
done

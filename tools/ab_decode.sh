# A/B of two builds in one GPU session: libecoserve.so (new) vs libecoserve_base.so (HEAD)
timeout 600 python -m pytest -q -x tests/test_gpu_ops.py -k "attention_decode" 2>&1 | tail -1
for i in 1 2 3; do
timeout 300 python tools/decode_ablate.py --one
ECOSERVE_LIB_AB=paper_2504_18154_b200/libecoserve_base.so timeout 300 python tools/decode_ablate.py --one
done

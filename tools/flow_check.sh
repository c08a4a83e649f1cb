for s in tiny-d128 tiny-gqa; do timeout 300 python tools/chain_diag.py $s 3 1e-2 | tail -1; done
timeout 900 python -m pytest -q -x tests/test_gpu_fullsize.py -k "single_gpu or sampled" tests/test_gpu_edge.py tests/test_gpu_instance.py 2>&1 | tail -2
for i in 1 2 3; do
timeout 300 python tools/decode_ablate.py --one
ECOSERVE_QKV_FUSE=0 timeout 300 python tools/decode_ablate.py --one
done

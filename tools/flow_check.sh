for s in tiny tiny-gqa tiny-d128; do timeout 300 python tools/chain_diag.py $s 3 1e-2 | tail -1; echo rc=$?; done
ECOSERVE_FLOW_TRACE=gpurun_out/flow_trace.txt timeout 300 python tools/decode_ablate.py --one; echo rc=$?
python tools/flow_trace.py gpurun_out/flow_trace.txt
timeout 600 python -m pytest -q -x tests/test_gpu_fullsize.py -k "single_gpu or sampled" 2>&1 | tail -3

ECOSERVE_GW_TRACE=gpurun_out/gw_trace.txt timeout 300 python tools/decode_ablate.py --one
python tools/gw_trace.py gpurun_out/gw_trace.txt

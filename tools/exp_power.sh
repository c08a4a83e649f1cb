# SM clock / power / throttle reasons while the 8B decode phase runs alone (decode_ablate) and
# while the 70B shard decodes
mkdir -p gpurun_out
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,utilization.gpu --format=csv -lms 100 > gpurun_out/power_decode.csv &
SMI=$!
sleep 1
for i in 1 2 3; do timeout 300 python tools/decode_ablate.py --one; done > gpurun_out/power_decode.jsonl 2>&1
kill $SMI
python - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/power_decode.csv")))[1:]
busy=[r for r in rows if len(r)>5 and r[5].strip().startswith(('9','10')) ]
import statistics as st
def f(x): return float(x.split()[0])
print("samples", len(rows), "busy", len(busy))
if busy:
    print("sm_mhz median", st.median(f(r[1]) for r in busy), "power median", st.median(f(r[2]) for r in busy),
          "power max", max(f(r[2]) for r in busy), "sw_power_cap active", sum('Active' == r[3].strip() for r in busy))
PY
cat gpurun_out/power_decode.jsonl

for i in 1 2; do
for b in 16 24 32 48; do
  echo "band=$b"; ECOSERVE_GEMM_BAND=$b python bench.py --steps 6 --warmup 3 --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(json.dumps({k:d.get(k) for k in ['value','prefill_tok_s','decode_tok_s','clocks']}))"
done
done

#!/bin/bash
# A/B: bench.py device timing (phase split) for each variant library.
for v in "$@"; do
  HBS_B200_LIB=tools/variants/$v.so python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['roofline']['phase_ms'].items()})"
done

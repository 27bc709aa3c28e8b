for c in 8 16 32; do
HBS_HOST_CHUNKS=$c timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('chunks $c', d['e2e']['s_per_step'], d['e2e']['value'])"
done

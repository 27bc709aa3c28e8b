mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_split3.json 2> gpurun_out/bench_split3.err
timeout 600 python bench.py --steps 10 --warmup 3 --n 1000000 --no-cpu-baseline --no-e2e > gpurun_out/bench_r02_c4_uneven.json 2> gpurun_out/bench_r02_c4_uneven.err
python -c "
import json
for f in ('bench_split3', 'bench_r02_c4_uneven'):
    d = json.loads(open('gpurun_out/' + f + '.json').read().strip().splitlines()[-1]); print(f, d['ms_per_step'], d['value'], d['gpu_launches'], d['roofline']['phase_ms'], d['e2e'] and d['e2e']['s_per_step'])
"

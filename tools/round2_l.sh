mkdir -p gpurun_out
timeout 300 python tools/dbg/sweep_hash.py > gpurun_out/hash_split.txt 2>&1; cat gpurun_out/hash_split.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_split.json 2> gpurun_out/bench_split.err
python -c "
import json
d = json.loads(open('gpurun_out/bench_split.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['gpu_launches'], d['roofline']['step_frac'], d['roofline']['frac'], d['roofline']['phase_ms'], d['e2e']['s_per_step'], d['accuracy'])"
timeout 300 python tools/dbg/level_phases.py > gpurun_out/level_phases_split.txt 2>&1; cat gpurun_out/level_phases_split.txt

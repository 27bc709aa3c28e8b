set -x
mkdir -p gpurun_out
timeout 300 python tools/dbg/sweep_hash.py > gpurun_out/hash_pipe2.txt 2>&1; cat gpurun_out/hash_pipe2.txt
timeout 300 python tools/dbg/pipe_trace.py > gpurun_out/trace_pipe2.txt 2>&1; cat gpurun_out/trace_pipe2.txt
timeout 300 python tools/dbg/level_phases.py > gpurun_out/level_phases_pipe2.txt 2>&1; cat gpurun_out/level_phases_pipe2.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pipe2.json 2> gpurun_out/bench_pipe2.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_pipe2.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['phase_ms'], d['accuracy'], d['roofline']['step_frac'])"

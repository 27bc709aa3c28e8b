set -x
mkdir -p gpurun_out
timeout 300 python tools/dbg/sweep_hash.py > gpurun_out/hash_pipe4.txt 2>&1; cat gpurun_out/hash_pipe4.txt
timeout 300 python tools/dbg/pipe_trace.py > gpurun_out/trace_pipe4.txt 2>&1; cat gpurun_out/trace_pipe4.txt
timeout 300 python tools/dbg/level_phases.py > gpurun_out/level_phases_pipe4.txt 2>&1; head -14 gpurun_out/level_phases_pipe4.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log

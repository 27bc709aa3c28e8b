mkdir -p gpurun_out
export HBS_SPLIT=1
timeout 300 python tools/dbg/sweep_hash.py > gpurun_out/hash_split.txt 2>&1; cat gpurun_out/hash_split.txt
timeout 300 python tools/dbg/split_trace.py > gpurun_out/trace_split.txt 2>&1; cat gpurun_out/trace_split.txt
N=262144 timeout 300 python tools/dbg/level_phases.py > gpurun_out/level_phases_split.txt 2>&1; head -3 gpurun_out/level_phases_split.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_size.py -m gpu -x -q > gpurun_out/pytest_split.log 2>&1; tail -4 gpurun_out/pytest_split.log

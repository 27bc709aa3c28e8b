mkdir -p gpurun_out
export HBS_SPLIT=1
timeout 300 python tools/dbg/split_trace.py > gpurun_out/trace_split.txt 2>&1; sed -n 8,14p gpurun_out/trace_split.txt
N=262144 timeout 300 python tools/dbg/level_phases.py > gpurun_out/level_phases_split.txt 2>&1; head -3 gpurun_out/level_phases_split.txt

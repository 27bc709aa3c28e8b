# traces + launch lists for the two probe paths
set -x
mkdir -p gpurun_out
export HBS_B200_LIB=tools/variants/hbs_trace.so
timeout 300 python tools/trace/run_trace.py > gpurun_out/trace_fused.txt 2>&1
timeout 300 python tools/dbg/gram_tm_trace.py > gpurun_out/trace_gram_tm.txt 2>&1
HBS_GRAM=1 timeout 300 python tools/trace/run_trace.py > gpurun_out/trace_pre.txt 2>&1
unset HBS_B200_LIB
KF='regex:probe_fused|hqr_kernel|bgemm|cholqr|rinv_blocks|applyq|fill_log|gram'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KF" --csv --log-file gpurun_out/launches_default.csv python tools/profile_level.py --n 65536 --reps 1 > gpurun_out/ncu_launch.log 2>&1
HBS_GRAM=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KF" --csv --log-file gpurun_out/launches_gram.csv python tools/profile_level.py --n 65536 --reps 1 > gpurun_out/ncu_launch_g.log 2>&1
python tools/dbg/ll_sum.py gpurun_out/launches_default.csv
python tools/dbg/ll_sum.py gpurun_out/launches_gram.csv

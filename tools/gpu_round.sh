# One GPU round: tests, smoke, bench (N=1), launch list of this library's kernels, full ncu of the top kernels.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "reference rc=$?"
KF='regex:probe_fused|hqr_kernel|bgemm|cholqr|rinv_blocks|applyq|fill_log|gram'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KF" --csv --log-file gpurun_out/launches.csv python tools/profile_level.py --n 65536 --reps 1 > gpurun_out/ncu_launch.log 2>&1
python tools/dbg/ll_sum.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:probe_fused_split -c 1 -o gpurun_out/fused python tools/profile_level.py --n 65536 --reps 1 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cholqr -c 1 -o gpurun_out/cholqr python tools/profile_level.py --n 65536 --reps 1 >> gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bgemm -s 20 -c 1 -o gpurun_out/bgemm python tools/profile_level.py --n 65536 --reps 1 >> gpurun_out/ncu_full.log 2>&1

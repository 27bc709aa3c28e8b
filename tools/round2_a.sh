# Round-2 status run: tests, bench on both probe paths, per-level phases.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
HBS_GRAM=1 timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_gram.json 2> gpurun_out/bench_gram.err
timeout 300 python tools/dbg/level_phases.py > gpurun_out/level_phases_default.txt 2>&1
HBS_GRAM=1 timeout 300 python tools/dbg/level_phases.py > gpurun_out/level_phases_gram.txt 2>&1
tail -3 gpurun_out/pytest_gpu.log

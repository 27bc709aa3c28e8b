set -x
mkdir -p gpurun_out
HBS_PIPE=0 timeout 300 python tools/dbg/sweep_hash.py > gpurun_out/hash_oneshot.txt 2>&1
timeout 300 python tools/dbg/sweep_hash.py > gpurun_out/hash_pipe.txt 2>&1
cat gpurun_out/hash_oneshot.txt gpurun_out/hash_pipe.txt
timeout 300 python tools/dbg/level_phases.py > gpurun_out/level_phases_pipe.txt 2>&1
cat gpurun_out/level_phases_pipe.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pipe.json 2> gpurun_out/bench_pipe.err
tail -c 1500 gpurun_out/bench_pipe.json

mkdir -p gpurun_out
KF='regex:probe_fused|gram'
for v in hbs_trace pairs_trace; do
HBS_GRAM=1 HBS_B200_LIB=tools/variants/$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KF" --csv --log-file gpurun_out/ll_$v.csv python tools/profile_level.py --n 65536 --reps 1 > gpurun_out/ncu_ll_$v.log 2>&1
echo $v; python tools/dbg/ll_sum.py gpurun_out/ll_$v.csv | head -4
grep -m3 "probe_fused_kernel<6, 1, 128, 192, 1>\|gram_factor_tm" gpurun_out/ll_$v.csv | cut -c1-200
done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02_c4.json 2> gpurun_out/bench_r02_c4.err; tail -c 600 gpurun_out/bench_r02_c4.json
timeout 600 python bench.py --steps 5 --warmup 3 --n 1000000 --no-cpu-baseline --no-e2e > gpurun_out/bench_r02_c4_uneven.json 2> gpurun_out/bench_r02_c4_uneven.err; python -c "
import json
for f in ('bench_r02_c4', 'bench_r02_c4_uneven'):
    d = json.loads(open('gpurun_out/' + f + '.json').read().strip().splitlines()[-1]); print(f, d['ms_per_step'], d['value'], d['roofline']['phase_ms'], d['e2e'], d['cpu_baseline'] and d['cpu_baseline']['value'])
"

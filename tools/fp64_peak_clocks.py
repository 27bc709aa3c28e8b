"""FP64 roofline denominator with a clock record: runs tools/fp64_peak (DMMA /
DFMA microbenchmark, built from tools/fp64_peak.cu) and tools/dgemm_peak.py
(cuBLAS DGEMM) repeatedly for ~10 s while nvidia-smi samples SM clocks and
throttle reasons; writes profiles/fp64_peaks_r02.json.
python tools/fp64_peak_clocks.py"""
import json, os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ClockSampler

HERE = os.path.dirname(os.path.abspath(__file__))
binp = os.path.join(HERE, "fp64_peak")
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", binp,
                os.path.join(HERE, "fp64_peak.cu")], check=True)
runs = []
with ClockSampler(0) as clocks:
    t0 = time.time()
    while time.time() - t0 < 8.0:
        runs.append(json.loads(subprocess.run([binp], capture_output=True, text=True, check=True).stdout))
    dg = json.loads(subprocess.run([sys.executable, os.path.join(HERE, "dgemm_peak.py")], capture_output=True,
                                   text=True, check=True).stdout)
best = {}
for r in runs:
    for k, v in r.items():
        if isinstance(v, (int, float)) and k != "sms":
            best[k] = max(best.get(k, 0.0), v)
out = {"gpu": runs[0]["gpu"], "sms": runs[0]["sms"], "repeats": len(runs), **best, **dg}
dmma = max(v for k, v in best.items() if k.startswith("dmma"))
out["fp64_peak_tflops"] = dmma
out["fp64_spec_tflops"] = 40.0
out["clocks"] = clocks.summary()
out["note"] = ("round 2: best of repeated runs of tools/fp64_peak.cu (DMMA m8n8k4 / m16n8k4 / m16n8k16 and DFMA) "
               "and tools/dgemm_peak.py (cuBLAS DGEMM) with nvidia-smi clocks sampled throughout; roofline "
               "denominator = max DMMA figure; the NVIDIA spec figure (40 TF) is quoted beside it")
path = os.path.join(os.path.dirname(HERE), "profiles", "fp64_peaks_r02.json")
with open(path, "w") as fh:
    json.dump(out, fh, indent=1)
print(json.dumps({k: out[k] for k in ("fp64_peak_tflops", "clocks", "dgemm_8192_tflops")}))

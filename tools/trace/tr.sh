# Fused-kernel and CholeskyQR2 clock64 traces of one c4-shaped level (CTA 0),
# with the tracing library built by build_trace.sh (EXTRA="-DPF_TRACE_J0=32" traces panel 1).
python tools/trace/run_trace.py > gpurun_out/trace_fused.txt 2>&1
python tools/trace/run_cq_trace.py > gpurun_out/trace_cholqr.txt 2>&1

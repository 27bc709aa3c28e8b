python tools/trace/run_trace.py > gpurun_out/trace0.txt 2>&1
cp tools/trace/_t32.so tools/trace/_hbs_b200_trace.so
python tools/trace/run_trace.py > gpurun_out/trace32.txt 2>&1

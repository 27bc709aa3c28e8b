mkdir -p gpurun_out
export N=262144
echo base; python tools/dbg/level_phases.py | head -2
for v in fr frd sl frsl; do echo $v; HBS_B200_LIB=tools/variants/$v.so python tools/dbg/level_phases.py | head -2; done

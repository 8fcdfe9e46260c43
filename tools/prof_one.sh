# ncu --set full capture (with source) of one kernel of one config: bash tools/prof_one.sh <kernel regex> <config> <out name> [lib variant]
lib=$PWD/paper_1203_0889_b200/lib/libfmm_b200.so; [ -n "$4" ] && lib=$PWD/paper_1203_0889_b200/lib/libfmm_b200_$4.so
FMM_B200_LIB=$lib ncu --set full --clock-control none --import-source on -k regex:$1 -c 1 -o gpurun_out/$3 -f \
  python tools/profile_step.py --config $2 --warmup 0 --steps 1 > gpurun_out/ncu_$3.log 2>&1
tail -2 gpurun_out/ncu_$3.log

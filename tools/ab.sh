# A/B of library variants lib/libfmm_b200_<v>.so ("main" = the default build) over configs:
#   bash tools/ab.sh "C2 C3 C5" main base nosleep
# prints the last-step stage times (serialised stages: kernel times are the kernels alone) and
# the default-overlap step time, averaged over 10 steps
cfgs=$1; shift
for v in "$@"; do
  lib=$PWD/paper_1203_0889_b200/lib/libfmm_b200_$v.so; [ $v = main ] && lib=$PWD/paper_1203_0889_b200/lib/libfmm_b200.so
  for cfg in $cfgs; do
    s=$(FMM_B200_LIB=$lib python tools/profile_step.py --config $cfg --warmup 3 --steps 10 --serial 2>&1 | head -1)
    o=$(FMM_B200_LIB=$lib python tools/profile_step.py --config $cfg --warmup 3 --steps 10 2>&1 | head -1)
    echo "$v $cfg serial: $(echo $s | grep -oE "'(p2p_kernel_ms|m2l_kernel_ms|traverse_ms|total_ms)': [0-9.]*" | tr '\n' ' ') | overlap total: $(echo $o | grep -oE "'total_ms': [0-9.]*")"
  done
done

# P2P kernel ms of narrow-CTA variants (FMM_P2P_SMALL=1) for the given library variants on C3 / C5
for v in "$@"; do
  lib=$PWD/paper_1203_0889_b200/lib/libfmm_b200_$v.so; [ $v = main ] && lib=$PWD/paper_1203_0889_b200/lib/libfmm_b200.so
  for cfg in C3 C5; do
    r=$(FMM_B200_LIB=$lib FMM_P2P_SMALL=1 python tools/profile_step.py --config $cfg --warmup 3 --steps 10 --serial 2>&1 | head -1)
    echo "$v small=1 $cfg $(echo $r | grep -oE "'(p2p_kernel_ms)': [0-9.]*" | tr '\n' ' ')"
  done
done

# A/B of p >= 7 M2L variants: M2L stage ms (serial stages) on C5 (p = 10) and a C4-shaped N = 2M
# p = 8 case; "main" = the default build. Then the C5/C4-shape parity tests on the first variant.
for v in "$@"; do
  lib=$PWD/paper_1203_0889_b200/lib/libfmm_b200_$v.so; [ $v = main ] && lib=$PWD/paper_1203_0889_b200/lib/libfmm_b200.so
  for cfg in "C5" "C4 --n 2097152"; do
    r=$(FMM_B200_LIB=$lib timeout 300 python tools/profile_step.py --config $cfg --warmup 2 --steps 5 --serial 2>&1 | head -1)
    echo "$v $cfg $(echo $r | grep -oE "'(m2l_kernel_ms|m2l_ms)': [0-9.]*" | tr '\n' ' ')"
  done
done

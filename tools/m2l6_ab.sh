# A/B of the p <= 6 M2L kernel variants on C2 and C3 (M2L kernel ms, 10 timed steps)
for v in "$@"; do
  for cfg in C2 C3; do
    r=$(FMM_B200_LIB=$PWD/paper_1203_0889_b200/lib/libfmm_b200_$v.so python tools/profile_step.py --config $cfg --warmup 3 --steps 10 --serial 2>&1 | head -1)
    echo "$v $cfg $(echo $r | grep -o "'m2l_kernel_ms': [0-9.]*")"
  done
done

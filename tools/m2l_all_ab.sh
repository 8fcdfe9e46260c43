# M2L stage ms (serial stages) for library variants over C1 C2 C3 C5 and a C4-shaped N = 2M p = 8 case
for v in "$@"; do
  lib=$PWD/paper_1203_0889_b200/lib/libfmm_b200_$v.so; [ $v = main ] && lib=$PWD/paper_1203_0889_b200/lib/libfmm_b200.so
  for cfg in "C1" "C2" "C3" "C5" "C4 --n 2097152"; do
    r=$(FMM_B200_LIB=$lib timeout 300 python tools/profile_step.py --config $cfg --warmup 2 --steps 5 --serial 2>&1 | head -1)
    echo "$v $cfg $(echo $r | grep -oE "'(m2l_kernel_ms|m2l_ms)': [0-9.]*" | tr '\n' ' ')"
  done
done

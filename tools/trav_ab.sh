# A/B of traversal variants: traverse-stage ms on C1 / C2 / C3 / C5 (10 steps, default overlap); "main" = default build
for v in "$@"; do
  lib=$PWD/paper_1203_0889_b200/lib/libfmm_b200_$v.so; [ $v = main ] && lib=$PWD/paper_1203_0889_b200/lib/libfmm_b200.so
  for cfg in ${TRAV_CFGS:-C1 C2 C3 C5}; do
    r=$(FMM_B200_LIB=$lib timeout 120 python tools/profile_step.py --config $cfg --warmup 3 --steps 10 2>&1 | head -1)
    echo "$v $cfg $(echo $r | grep -o "'traverse_ms': [0-9.]*") $(echo $r | grep -o "'total_ms': [0-9.]*")"
  done
done

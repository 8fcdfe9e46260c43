# A/B of P2P library variants (lib/libfmm_b200_<v>.so): P2P kernel ms on C2 / C3 / C5 (10 steps)
for v in "$@"; do
  for cfg in C2 C3 C5; do
    r=$(FMM_B200_LIB=$PWD/paper_1203_0889_b200/lib/libfmm_b200_$v.so python tools/profile_step.py --config $cfg --warmup 3 --steps 10 --serial 2>&1 | head -1)
    echo "$v $cfg $(echo $r | grep -o "'p2p_kernel_ms': [0-9.]*")"
  done
done

# A/B of p = 10 M2L variants on C5 (M2L kernel ms, serial stages) + the C5-shape parity test
for v in "$@"; do
  r=$(FMM_B200_LIB=$PWD/paper_1203_0889_b200/lib/libfmm_b200_$v.so timeout 200 python tools/profile_step.py --config C5 --warmup 2 --steps 3 --serial 2>&1 | head -1)
  echo "$v C5 $(echo $r | grep -o "'m2l_kernel_ms': [0-9.]*")"
done

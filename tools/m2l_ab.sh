# A/B of M2L library variants (lib/libfmm_b200_<v>.so): M2L kernel time on C2 (p=6), C5 (p=10)
# and a C4-shaped N=2M p=8 case, plus the parity tests.
for v in "$@"; do
  for cfg in "C2" "C5" "C4 --n 2097152"; do
    r=$(FMM_B200_LIB=$PWD/paper_1203_0889_b200/lib/libfmm_b200_$v.so python tools/profile_step.py --config $cfg --warmup 2 --steps 3 --serial 2>&1 | head -1)
    echo "$v $cfg $(echo $r | grep -o "'m2l_kernel_ms': [0-9.]*")"
  done
  FMM_B200_LIB=$PWD/paper_1203_0889_b200/lib/libfmm_b200_$v.so python -m pytest tests/test_gpu_parity.py -q -x -k "pipeline_vs_oracle or fixtures" 2>&1 | tail -1
done

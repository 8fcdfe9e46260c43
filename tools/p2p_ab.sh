for v in old ws6 ws5; do
  for cfg in C2 C3 C5; do
    r=$(FMM_B200_LIB=$PWD/paper_1203_0889_b200/lib/libfmm_b200_$v.so python tools/profile_step.py --config $cfg --warmup 3 --steps 5 --serial 2>&1 | head -1)
    echo "$v $cfg $(echo $r | grep -o "'p2p_kernel_ms': [0-9.]*")"
  done
done
FMM_B200_LIB=$PWD/paper_1203_0889_b200/lib/libfmm_b200_ws6.so python -m pytest tests/test_gpu_parity.py -q -x -k "pipeline_vs_oracle or fixtures or deterministic" 2>&1 | tail -2
FMM_B200_LIB=$PWD/paper_1203_0889_b200/lib/libfmm_b200_ws5.so python -m pytest tests/test_gpu_parity.py -q -x -k "pipeline_vs_oracle or fixtures or deterministic" 2>&1 | tail -2

#!/bin/bash
# Times the M2L kernel of each library variant (lib/libfmm_b200*.so) on C2 and C3.
for lib in paper_1203_0889_b200/lib/libfmm_b200*.so; do
  for cfg in C2 C3; do
    r=$(FMM_B200_LIB=$PWD/$lib python tools/profile_step.py --config $cfg --warmup 3 --steps 3 --serial 2>&1 | head -1)
    echo "$(basename $lib) $cfg $(echo $r | grep -o "'m2l_kernel_ms': [0-9.]*")"
  done
done

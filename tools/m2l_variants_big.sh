#!/bin/bash
# Times the M2L kernel of each library variant on C5 (p=10) and a C4-shaped run (p=8, N=2M).
for lib in paper_1203_0889_b200/lib/libfmm_b200*.so; do
  r=$(FMM_B200_LIB=$PWD/$lib python tools/profile_step.py --config C5 --warmup 1 --steps 1 --serial 2>&1 | head -1)
  r4=$(FMM_B200_LIB=$PWD/$lib python tools/profile_step.py --config C4 --n 2097152 --warmup 1 --steps 1 --serial 2>&1 | head -1)
  echo "$(basename $lib) C5 $(echo $r | grep -o "'m2l_kernel_ms': [0-9.]*") C4s $(echo $r4 | grep -o "'m2l_kernel_ms': [0-9.]*")"
done

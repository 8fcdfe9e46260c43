# ncu --set full captures (with source) of the three kernels the verdict names, brought back as
# .ncu-rep for local analysis: M2L p=10 (C5), P2P (C5), k_step deepest levels (C3)
ncu --set full --clock-control none --import-source on -k regex:k_m2l_big2 -c 1 -o gpurun_out/m2l10_c5 -f \
  python tools/profile_step.py --config C5 --warmup 0 --steps 1 > gpurun_out/ncu_m2l10.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_p2p_fp32_ws -c 1 -o gpurun_out/p2p_c5 -f \
  python tools/profile_step.py --config C5 --warmup 0 --steps 1 > gpurun_out/ncu_p2p_c5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_m2l_reg -c 1 -o gpurun_out/m2l6_c2 -f \
  python tools/profile_step.py --config C2 --warmup 0 --steps 1 > gpurun_out/ncu_m2l6.log 2>&1
ls -la gpurun_out/*.ncu-rep

# Evidence refresh: bench launch list (C2), ncu --set full of M2L p=10 (C5) and the deepest k_step levels (C2)
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c2_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_m2l_big2 -c 1 -o /tmp/m2l10 \
  python tools/profile_step.py --config C5 --warmup 0 --steps 1 > gpurun_out/ncu_m2l10.log 2>&1
python tools/ncu_summary.py /tmp/m2l10.ncu-rep > gpurun_out/m2l10_summary.txt 2>&1
ncu --set full --clock-control none -k regex:k_step --launch-skip 15 -c 3 -o /tmp/kstep2 \
  python tools/profile_step.py --config C2 --warmup 1 --steps 1 > gpurun_out/ncu_kstep2.log 2>&1
python tools/ncu_summary.py /tmp/kstep2.ncu-rep > gpurun_out/kstep2_summary.txt 2>&1
ls -la gpurun_out

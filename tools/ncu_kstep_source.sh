ncu --set full --import-source on --clock-control none -k regex:k_step --launch-skip 48 -c 3 -o /tmp/ks3 python tools/profile_step.py --config C3 --warmup 1 --steps 1 > gpurun_out/ks3.log 2>&1
ncu -i /tmp/ks3.ncu-rep --page source --csv --print-source sass > gpurun_out/ks3_sass.csv 2>&1
python tools/ncu_summary.py /tmp/ks3.ncu-rep > gpurun_out/ks3_summary.txt 2>&1
ls -la gpurun_out/ks3*

# Traversal (k_step) evidence: stage times and launch list at C3, ncu sections of k_step at C3/C2
python tools/profile_step.py --config C3 --warmup 2 --steps 3 > gpurun_out/ps_c3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c3_now.csv python tools/profile_step.py --config C3 --warmup 1 --steps 1 > gpurun_out/ncu_l3.log 2>&1
S="--section SpeedOfLight --section MemoryWorkloadAnalysis --section WarpStateStats --section LaunchStats --section Occupancy --section SchedulerStats --section ComputeWorkloadAnalysis"
ncu $S --clock-control none -k regex:k_step --launch-skip 40 -c 26 -o /tmp/kstep_c3 python tools/profile_step.py --config C3 --warmup 2 --steps 1 > gpurun_out/ncu_ks.log 2>&1
ncu -i /tmp/kstep_c3.ncu-rep --page details --csv > gpurun_out/kstep_c3.csv
ncu $S --clock-control none -k regex:k_step --launch-skip 30 -c 18 -o /tmp/kstep_c2 python tools/profile_step.py --config C2 --warmup 2 --steps 1 > gpurun_out/ncu_ks2.log 2>&1
ncu -i /tmp/kstep_c2.ncu-rep --page details --csv > gpurun_out/kstep_c2.csv
ls -la gpurun_out

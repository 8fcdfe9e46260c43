# Round-2 evidence refresh (one B200): GPU tests, smoke, one bench line per config, reference arm,
# then (each only after the plain command exited 0) the ncu launch lists of the bench command at
# C2 / C5 and --set full captures of the top kernels. Summaries are written next to the reports.
set -x
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -n 2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -n 2 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err || exit 1
for c in C1 C3 C4 C5; do
  python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
for c in C2 C5; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_$c.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-fp64-mode > gpurun_out/ncu_bench_$c.log 2>&1
  python tools/launch_summary.py gpurun_out/launches_$c.csv > gpurun_out/launches_${c}_summary.txt 2>&1
done
cap() {  # kernel regex, config, name
  ncu --set full --clock-control none --import-source on -k regex:$1 -c 1 -o gpurun_out/$3 -f \
    python tools/profile_step.py --config $2 --warmup 0 --steps 1 > gpurun_out/ncu_$3.log 2>&1
  python tools/ncu_summary.py gpurun_out/$3.ncu-rep > gpurun_out/$3_summary.txt 2>&1
}
cap k_p2p_fp32_ws C2 r2f_p2p_c2
cap k_m2l_reg C2 r2f_m2l6_c2
cap k_m2l_flat C5 r2f_m2l10_c5
cap k_p2p_fp32_ws C5 r2f_p2p_c5
ls -la gpurun_out | head -60

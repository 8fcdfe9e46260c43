# One bench line per BASELINE config (C2 = the headline with its CPU baseline; the others without)
# into gpurun_out/bench_<cfg>.json, plus the GPU test suite.
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -n 2 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
for c in C1 C3 C4 C5; do
  python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
for c in C1 C2 C3 C4 C5; do
  python -c "
import json,sys
d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1])
print('$c', round(d['ms_per_step'],3), 'ms', '%.3e'%d['value'], 'e2e %.3e'%d['e2e']['value'], 'p2p frac %.3f'%d['roofline']['frac'], {k: round(v,3) for k,v in d['stage_ms'].items()})
" || tail -3 gpurun_out/bench_$c.err
done

#!/bin/bash
# DRAM bytes per launch of the P2P kernel at every BASELINE config (and the FP64 parity mode at C2),
# one ncu pass each over the first P2P launch of a short bench run (default cache control: L2
# flushed before the launch, as in the --set full capture). Output: gpurun_out/traffic_<cfg>.csv,
# folded into profiles/ncu_traffic.json by tools/p2p_traffic_fold.py.
set -u
mkdir -p gpurun_out
run() {  # config precision
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:'k_p2p_fp(32_ws|64)' -c 1 --csv \
    --log-file gpurun_out/traffic_$1_$2.csv \
    python bench.py --config $1 --precision $2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/traffic_$1_$2.log 2>&1
  echo "$1 $2 rc=$?"
}
for c in C1 C2 C3 C4 C5; do run $c fp32; done
run C2 fp64

# whole-step ms (default overlap) of library variants: bash tools/step_ab.sh "C2 C3" main other
cfgs=$1; shift
for v in "$@"; do
  lib=$PWD/paper_1203_0889_b200/lib/libfmm_b200_$v.so; [ $v = main ] && lib=$PWD/paper_1203_0889_b200/lib/libfmm_b200.so
  for cfg in $cfgs; do
    r=$(FMM_B200_LIB=$lib timeout 300 python tools/profile_step.py --config $cfg --warmup 3 --steps 10 2>&1 | head -1)
    echo "$v $cfg $(echo $r | grep -oE "'(total_ms|p2p_ms|downward_ms)': [0-9.]*" | tr '\n' ' ')"
  done
done

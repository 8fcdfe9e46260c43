# Stage overlap A/B on C2/C3/C5: level 1 (upward || traversal) vs level 2 (also M2L || P2P), with
# the P2P CTAs per SM capped by a dynamic shared-memory pad (FMM_P2P_PAD_KB).
for cfg in C2 C3 C5; do
  echo "$cfg L1 $(python tools/profile_step.py --config $cfg --warmup 3 --steps 10 --overlap-level 1 2>&1 | head -1 | grep -o "'total_ms': [0-9.]*")"
  for pad in 0 10 22; do
    echo "$cfg L2 pad$pad $(FMM_P2P_PAD_KB=$pad python tools/profile_step.py --config $cfg --warmup 3 --steps 10 --overlap-level 2 2>&1 | head -1 | grep -o "'total_ms': [0-9.]*")"
  done
done

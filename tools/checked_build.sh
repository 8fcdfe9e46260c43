#!/bin/bash
# Checked library (device bounds checks, FMM_CHECKS=1) as lib/libfmm_b200_checked.so, then the
# whole GPU test suite against it (FMM_B200_LIB); log: gpurun_out/checked_build.log.
# compute-sanitizer is refused on the GPU pool, so this run is the memory-safety evidence.
set -e
cd "$(dirname "$0")/.."
[ -f paper_1203_0889_b200/lib/libfmm_b200_checked.so ] || bash tools/build_variant.sh checked capi,tree_build,traverse,p2p,expansions,m2l,ops,shard,comm "-DFMM_CHECKS=1"
mkdir -p gpurun_out
set +e
FMM_B200_LIB=$PWD/paper_1203_0889_b200/lib/libfmm_b200_checked.so timeout 2400 python -m pytest tests -m gpu -q \
  --deselect tests/test_cpp_mirror.py > gpurun_out/checked_build.log 2>&1
echo "rc=$?" >> gpurun_out/checked_build.log
grep -c "FMM_CHECK failed" gpurun_out/checked_build.log >> gpurun_out/checked_build.log

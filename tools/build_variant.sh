# Builds lib/libfmm_b200_<name>.so with the given sources compiled with extra -D switches:
#   bash tools/build_variant.sh <name> <source stem[,stem...]> "-DFOO=1 -DBAR=2"
set -e
name=$1; srcs=$2; defs=$3
R=$(cd "$(dirname "$0")/.." && pwd)
make -s -C $R/paper_1203_0889_b200/csrc >/dev/null
V=$R/build/var_$name; mkdir -p $V
ARCH="-gencode arch=compute_100a,code=sm_100a"
for src in ${srcs//,/ }; do
  extra=""; [ "$src" = p2p ] && extra="-ftz=true"
  /usr/local/cuda/bin/nvcc $ARCH -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-O2 \
    -I$R/include $extra $defs -c $R/paper_1203_0889_b200/csrc/$src.cu -o $V/$src.o
done
objs=""
for o in capi tree_build traverse p2p expansions m2l ops shard comm; do
  if [[ ",$srcs," == *",$o,"* ]]; then objs="$objs $V/$o.o"; else objs="$objs $R/build/obj/$o.o"; fi
done
/usr/local/cuda/bin/nvcc $ARCH -shared -o $R/paper_1203_0889_b200/lib/libfmm_b200_$name.so $objs -lcudart -ldl

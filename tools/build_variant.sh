#!/bin/bash
# Build an experimental libeq4 variant: tools/build_variant.sh NAME [nvcc -D flags...]
# -> variants/libeq4_NAME.so ; select it at run time with EQ4_LIB=variants/libeq4_NAME.so
# REV=<git rev> builds the kernels as of that revision instead of the working tree.
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
src=$root/paper_1911_02079_b200/csrc
out=$root/variants
mkdir -p $out/obj_$name
if [ -n "$REV" ]; then
  tmp=$(mktemp -d)
  (cd $root && git archive "$REV" paper_1911_02079_b200/csrc include | tar -x -C $tmp)
  src=$tmp/paper_1911_02079_b200/csrc
fi
F="-O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr"
for f in $src/*.cu; do
  b=$(basename $f .cu)
  /usr/local/cuda/bin/nvcc $F "$@" -c -o $out/obj_$name/$b.o $f 2>/dev/null &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libeq4_$name.so $out/obj_$name/*.o
rm -rf $out/obj_$name ${tmp:-}
echo $out/libeq4_$name.so

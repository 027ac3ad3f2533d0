#!/bin/bash
# Build libocean_b200.so with extra nvcc defines into lib/variants/NAME.so
#   tools/build_variant.sh NAME -DOCN_FUSE_W=4 ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=paper_2503_03326_b200/lib/variants; mkdir -p $out /tmp/ocn_var_$name
objs=""
for f in paper_2503_03326_b200/csrc/*.cu; do
  o=/tmp/ocn_var_$name/$(basename $f .cu).o
  if [ "$(basename $f)" = "${VARIANT_SRC:-spectral.cu}" ]; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Iinclude "$@" -c $f -o $o
  else
    o=paper_2503_03326_b200/build/$(basename $f .cu).o
  fi
  objs="$objs $o"
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/$name.so $objs -lcudart_static -lrt -ldl -lpthread
echo $out/$name.so

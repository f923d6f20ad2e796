#!/bin/bash
# A/B builds: tools/build_variant.sh NAME "-DMACRO=..."  ->  variants/NAME.so
# (load with MFD_LIB=variants/NAME.so; the default library is untouched)
set -e
cd "$(dirname "$0")/.."
name=$1; flags=$2
P=paper_1406_7459_b200
d=variants/build_$name; mkdir -p $d
NV="/usr/local/cuda/bin/nvcc -O3 -std=c++20 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -diag-suppress 177"
for f in ${VARIANT_MAIN:-engine_f32} ${VARIANT_SRCS:-}; do $NV $flags -c $P/csrc/$f.cu -o $d/$f.o & done
wait
objs=""
for o in $P/build/*.o; do b=$(basename $o); [ -f $d/$b ] && objs="$objs $d/$b" || objs="$objs $o"; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/$name.so $objs -lcudart -lnccl
echo variants/$name.so

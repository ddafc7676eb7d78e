#!/bin/bash
# Build an experiment variant of libb2s.so with extra nvcc defines:
#   tools/build_variant.sh NAME -DKNOB=1 ...   -> paper_2602_08387_b200/csrc/build/var_NAME/libb2s.so
# (run it with B2S_LIB=<that path> to A/B against the default build)
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2602_08387_b200/csrc"
out=build/var_$name
mkdir -p $out
ARCH="-gencode arch=compute_100a,code=sm_100a"
for f in *.cu; do
  nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I../../include "$@" \
       -c $f -o $out/${f%.cu}.o &
done
for f in *.cpp; do g++ -O3 -std=c++17 -fPIC -pthread -I../../include -c $f -o $out/${f%.cpp}.o & done
wait
nvcc $ARCH -shared -o $out/libb2s.so $out/*.o -lcuda -ldl -Xcompiler -pthread
echo $PWD/$out/libb2s.so

# Build an experimental / debug copy of the library: bash scripts/build_variant.sh NAME [-DFLAG ...]
# -> paper_1807_05358_b200/_lib/NAME/libparasim_cuda.so (select with PARASIM_B200_LIB)
set -e
name=$1; shift
out=paper_1807_05358_b200/_lib/$name
mkdir -p $out
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 \
  -Xcompiler -fPIC -shared -Iinclude "$@" -o $out/libparasim_cuda.so paper_1807_05358_b200/csrc/parasim_cuda.cu

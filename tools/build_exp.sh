# build experiment variants of the engine: tools/build_exp.sh NAME -DFLAG ...
# (paper_2007_06483_b200/_lib/exp/NAME.so; select with MTB_LIB_PATH)
set -e
name=$1; shift
mkdir -p paper_2007_06483_b200/_lib/exp
cd paper_2007_06483_b200/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr "$@" -shared -o ../_lib/exp/$name.so capi.cu pyramid.cu k1_rgb.cu threshold.cu search.cu shift.cu pipe.cu cluster.cu

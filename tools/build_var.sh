# Build a variant of libevd.so for an A/B (tools/ab_libs.sh):
#   bash tools/build_var.sh NAME [-DFLAG=...]...   ->  build_var/NAME.so
set -e
cd "$(dirname "$0")/.."
mkdir -p build_var
name=$1; shift
C=paper_2209_13168_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --fmad=false \
    -Xcompiler -fPIC,-ffp-contract=off -Xptxas -v --expt-relaxed-constexpr "$@" -shared \
    -o build_var/$name.so $C/evd_api.cu $C/evd_kernels.cu $C/evd_io.cu $C/evd_frontier_tiles.cu \
    2> build_var/$name.ptxas.log || { grep -i error build_var/$name.ptxas.log; exit 1; }
grep -A1 "k_solve_specILi512" build_var/$name.ptxas.log | grep -o "[0-9]* bytes spill stores.*\|Used [0-9]* registers" | head -2

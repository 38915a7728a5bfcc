# build a variant of the native library: tools/build_variant.sh NAME [-DFLAG ...] -> lib/libvar_NAME.so
# (select it at run time with SL_LIB_PATH=paper_2505_23022_b200/lib/libvar_NAME.so)
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2505_23022_b200"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -shared "$@" -I../include -o lib/libvar_$name.so csrc/sim_kernel.cu csrc/plan_kernels.cu csrc/predict_kernel.cu csrc/report_kernel.cu

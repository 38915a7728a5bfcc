# profiling build of the library with the one-CTA-per-segment phase stamps (tools/large_prof.py)
cd "$(dirname "$0")/../paper_2505_23022_b200" && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -shared -DSL_LARGE_PROF -I../include -o lib/libvar_lprof.so csrc/sim_kernel.cu csrc/plan_kernels.cu csrc/predict_kernel.cu csrc/report_kernel.cu

# per-phase cycle accounting of the sweep kernel (libvar_prof.so, tools/build_variant.sh prof -DSL_PHASE_PROF)
mkdir -p gpurun_out
SL_LIB_PATH=paper_2505_23022_b200/lib/libvar_prof.so timeout 600 python tools/phase_prof.py > gpurun_out/phase_prof.txt 2>&1; cat gpurun_out/phase_prof.txt

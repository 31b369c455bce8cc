#!/bin/bash
# production build + a tuning build of gemm.cu (RFK_GEMM_TUNING=1: timing experiments, RFK_GEMM_DBG timelines)
# linked into build/ab/lib_tune.so; select it with RF_LIB_PATH=build/ab/lib_tune.so (tools/gemm_probe.py etc.)
set -e
python -m paper_1808_00079_b200.build >/dev/null
mkdir -p build/ab
cp paper_1808_00079_b200/libreforward_b200.so build/ab/lib_new.so
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude -Ipaper_1808_00079_b200/csrc -diag-suppress 177,550,128 -DRFK_GEMM_TUNING=1 -c paper_1808_00079_b200/csrc/kernels/gemm.cu -o build/ab/gemm_tune.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/ab/lib_tune.so $(ls build/obj/*.o | grep -v "kernels__gemm.cu.o") build/ab/gemm_tune.o -ldl

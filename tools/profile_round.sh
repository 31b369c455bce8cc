#!/bin/bash
# Profiles of one round (run on the GPU box): bash tools/profile_round.sh r2
tag=${1:-r2}
o=gpurun_out/prof_$tag
mkdir -p $o
# 1. launch list with DRAM traffic of one eager ResNet-50 step
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $o/traffic.csv python tools/profile_step.py > /dev/null 2>&1
# 2. full captures of the top GEMM family and the BN backward kernels (a few launches each)
ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 40 -c 6 \
    -o $o/gemm_full python tools/profile_step.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:bn_bwd -s 4 -c 6 \
    -o $o/bn_full python tools/profile_step.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm_band|maxpool" -c 6 \
    -o $o/band_pool_full python tools/profile_step.py > /dev/null 2>&1
# 3. per-GEMM and per-instruction breakdowns (CUDA events, no profiler)
python tools/gemm_breakdown.py reforward resnet50 32 224 > $o/gemm_breakdown.txt 2>&1
python tools/step_breakdown.py resnet50 reforward 32 224 > $o/step_breakdown.txt 2>&1
# 4. ablation bounds (what removing each BN kernel family would save)
for m in 0 1 2 4 8 16 31; do RFK_ABLATE=$m python tools/ablate_time.py | tail -1; done > $o/ablation.txt 2>&1
ls -la $o

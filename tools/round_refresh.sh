#!/bin/bash
# One round refresh on the GPU box: GPU tests, a bench line of every BASELINE network, profiles.
#   gpurun -- bash tools/round_refresh.sh <tag>;  then here: python tools/update_profiles.py <tag>
tag=${1:-r2b}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_$tag.log 2>&1; echo "pytest rc $?" >> gpurun_out/gpu_tests_$tag.log
bash tools/bench_all.sh $tag > gpurun_out/bench_all_$tag.txt 2>&1
bash tools/profile_round.sh $tag > gpurun_out/profile_$tag.txt 2>&1
tail -3 gpurun_out/gpu_tests_$tag.log; cat gpurun_out/bench_all_$tag.txt

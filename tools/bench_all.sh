#!/bin/bash
# Round bench lines of every BASELINE network (run on the GPU box):
#   bash tools/bench_all.sh <tag>   ->  gpurun_out/bench_<tag>/<arch>_b<batch>_<hw>.json
tag=${1:-r2}
out=gpurun_out/bench_$tag
mkdir -p $out
run() {  # arch batch hw
  python bench.py --arch $1 --batch $2 --hw $3 --steps 20 --warmup 5 > $out/$1_b$2_$3.json 2> $out/$1_b$2_$3.err
  echo "$1 b$2 $3: $(python -c "import json;d=json.load(open('$out/$1_b$2_$3.json'));print(round(d['value']),'img/s e2e',round(d['e2e']['value']),'store-all',round(d['store_all']['value']),'overhead',round(d['overhead_vs_store_all'],3),'cut',round(d['memory']['cut_percent'],1),'frac',round(d['roofline']['frac'],3))" 2>&1 | tail -1)"
}
run resnet50 32 224
run resnet101 32 224
run vgg16 32 224
run alexnet 32 224
run densenet121 32 224
run inception_v3 32 299
run densenet121 64 600
run inception_v3 64 600

# batched-decode sweep (8-layer 7B stack); args: tag, then batch sizes
tag=$1; shift
for B in "$@"; do python bench.py --batch $B --layers 8 --steps 200 --warmup 20 --no-cpu-baseline --no-dense > gpurun_out/${tag}_B$B.json 2>gpurun_out/${tag}_B$B.err; python -c "import json;d=json.load(open('gpurun_out/${tag}_B$B.json'));print('$tag',$B,round(d['value']),round(d['per_layer_us'],1),round(d['roofline']['frac'],3))"; done

# A/B of programmatic dependent launch in the batched path (SG_PDL=1 vs plain launches)
python -m pytest tests -m gpu -x -q > gpurun_out/tgpu.log 2>&1; tail -2 gpurun_out/tgpu.log
for B in 5 8 16 32 64; do for P in 0 1; do SG_PDL=$((1-P)) python bench.py --batch $B --layers 8 --steps 200 --warmup 20 --no-cpu-baseline --no-dense > gpurun_out/pdl_B${B}_$P.json 2>gpurun_out/pdl_B${B}_$P.err; python -c "import json;d=json.load(open('gpurun_out/pdl_B${B}_$P.json'));print($B,'nopdl' if $P else 'pdl',round(d['value']),round(d['per_layer_us'],1),round(d['roofline']['frac'],3))"; done; done

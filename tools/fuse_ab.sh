# A/B of the batched-path fusions (SG_BATCH_FUSE bits: 1 compaction in gate_epi, 2 T reduce in t_kernel)
SG_BATCH_FUSE=3 python -m pytest tests/test_gpu_batch.py -x -q 2>&1 | tail -1
SG_BATCH_FUSE=1 python -m pytest tests/test_gpu_batch.py -x -q 2>&1 | tail -1
for B in 5 8 16; do for F in 0 1 2 3 0 3; do SG_BATCH_FUSE=$F python bench.py --batch $B --layers 8 --steps 300 --warmup 20 --no-cpu-baseline --no-dense > gpurun_out/fab_B${B}_$F.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/fab_B${B}_$F.json'));print($B,'fuse$F',round(d['value']),round(d['per_layer_us'],1))"; done; done

#!/bin/bash
# Round-2 evidence on one B200: GPU tests, smoke, headline + config bench lines, the
# reference arm, and the 32-layer batched sweep (sparse + dense comparator). Outputs
# under gpurun_out/ (copied to profiles/ by hand).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/tests_gpu_r02.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/tests_gpu_r02.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r02.log 2>&1; tail -3 gpurun_out/smoke_r02.log
for c in 7b mistral 13b; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_r02_$c.json 2> gpurun_out/bench_r02_$c.err
  python -c "import json; d=json.loads(open('gpurun_out/bench_r02_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['value'],1), d['unit'], 'e2e', round(d['e2e']['value'],1), 'frac', round(d['roofline']['frac'],3), 'us/layer', round(d.get('per_layer_us', 0),1))" || tail -3 gpurun_out/bench_r02_$c.err
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_r02_reference.json 2> gpurun_out/bench_r02_reference.err; tail -c 400 gpurun_out/bench_r02_reference.json
for B in 2 4 8 16 32 48 64; do
  timeout 600 python bench.py --batch $B --layers 32 --steps 50 --warmup 5 > gpurun_out/batch_r02_B$B.json 2> gpurun_out/batch_r02_B$B.err
  python -c "import json; d=json.loads(open('gpurun_out/batch_r02_B$B.json').read().strip().splitlines()[-1]); print('B=$B', 'tok/s %.0f us/layer %.1f frac %.3f | dense us/layer %.1f | sparse/dense %.2f | e2e %.0f' % (d['value'], d['per_layer_us'], d['roofline']['frac'], d['dense']['per_layer_us'], d['dense']['sparse_speedup'], d['e2e']['value']))" || tail -3 gpurun_out/batch_r02_B$B.err
done
for c in 13b mistral; do
  for B in 8 32; do
    timeout 600 python bench.py --config $c --batch $B --steps 30 --warmup 5 > gpurun_out/batch_r02_${c}_$B.json 2> gpurun_out/batch_r02_${c}_$B.err
    python -c "import json; d=json.loads(open('gpurun_out/batch_r02_${c}_$B.json').read().strip().splitlines()[-1]); print('$c B=$B', 'us/layer %.1f | dense %.1f | sparse/dense %.2f' % (d['per_layer_us'], d['dense']['per_layer_us'], d['dense']['sparse_speedup']))" || tail -3 gpurun_out/batch_r02_${c}_$B.err
  done
done

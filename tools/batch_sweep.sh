#!/bin/bash
# Batched-decode sweep (configs[4]): one JSON line per B (sparse tcgen05 path, dense
# comparator, e2e, roofline; layers chained through the residual stream, bench
# default --chain 2) into gpurun_out/batch_B*.json.
#   tools/batch_sweep.sh [layers] [B ...]     (default: the full 32-layer 7B stack)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
L=${1:-32}; shift
for B in ${@:-2 4 8 16 32 64}; do
  python bench.py --batch $B --layers $L --steps 50 --warmup 5 > gpurun_out/batch_B$B.json 2> gpurun_out/batch_B$B.err
  python -c "import json; d=json.loads(open('gpurun_out/batch_B$B.json').read().strip().splitlines()[-1]); print('B=$B', 'tok/s %.0f us/layer %.1f frac %.3f | dense us/layer %.1f | sparse/dense %.2f | e2e %.0f | %s' % (d['value'], d['per_layer_us'], d['roofline']['frac'], d['dense']['per_layer_us'], d['dense']['sparse_speedup'], d['e2e']['value'], d['config']['chain']))" || tail -5 gpurun_out/batch_B$B.err
done

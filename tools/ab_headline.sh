#!/bin/bash
# A/B of headline-kernel variants on the 7B 32-layer stack (residual chain):
# each SG_LIB variant (libsparsegate_b200_<v>.so; "" = the default build) twice,
# alternating, into gpurun_out/ab_<v>_<rep>.json; then the phase profile of the default.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
  for v in "" ${@}; do
    SG_LIB=$v python bench.py --steps 400 --warmup 20 --no-cpu-baseline --no-dense --no-diag \
      > gpurun_out/ab_${v:-default}_$rep.json 2> gpurun_out/ab_${v:-default}_$rep.err
  done
done
python tools/phase_profile.py --config 7b --layers 8 > gpurun_out/phases.txt 2>&1
for f in gpurun_out/ab_*.json; do
  python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['per_layer_us'],2), 'unchained', round(d['unchained']['per_layer_us'],2))"
done

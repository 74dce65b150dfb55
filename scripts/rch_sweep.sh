#!/bin/bash
# Rows-per-tile sweep (SWDFT2D_K1_RCH override) for one config: bench.py kernel-only lines.
#   bash scripts/rch_sweep.sh c2 fp32 "497 249 166 125 100 83 71 62 50 40"
cfg=$1; prec=$2; shift 2
for r in $1; do
  SWDFT2D_K1_RCH=$r python bench.py --config $cfg --precision $prec --steps 10 --warmup 3 \
    --no-cpu --no-e2e --no-others | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'config': '$cfg', 'prec': '$prec', 'rch': $r, 'gcoef_s': l['value']/1e9, 'frac': l['roofline']['frac']}))"
done
python bench.py --config $cfg --precision $prec --steps 10 --warmup 3 --no-cpu --no-e2e --no-others | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'config': '$cfg', 'prec': '$prec', 'rch': 'model', 'gcoef_s': l['value']/1e9, 'frac': l['roofline']['frac']}))"

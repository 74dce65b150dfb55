#!/bin/bash
# K1 persistent vs one-shot grid (SWDFT2D_K1_ONESHOT) over rows-per-tile (SWDFT2D_K1_RCH)
# writes one JSON line per run to $OUT
OUT=${OUT:-gpurun_out/oneshot_sweep.jsonl}
: > $OUT
for cfg in ${CFGS:-c4 c2 c3 c5}; do
  for prec in ${PRECS:-fp32}; do
    run() {  # $1 oneshot $2 rch
      line=$(SWDFT2D_K1_ONESHOT=$1 SWDFT2D_K1_RCH=$2 timeout 300 python bench.py --config $cfg --precision $prec \
             --no-cpu --no-e2e --no-others --steps 10 --warmup 3 2>/dev/null | tail -1)
      python - "$cfg" "$prec" "$1" "$2" "$line" >> $OUT <<'PY'
import json, sys
cfg, prec, one, rch, line = sys.argv[1:]
try:
    d = json.loads(line)
    print(json.dumps({"config": cfg, "prec": prec, "oneshot": int(one), "rch": int(rch),
                      "gcoef_s": round(d["value"] / 1e9, 1), "write_tbs": round(d["hbm_write_gbs"] / 1e3, 3),
                      "ms": round(d["ms_per_step"], 4)}))
except Exception as e:
    print(json.dumps({"config": cfg, "prec": prec, "oneshot": int(one), "rch": int(rch), "error": str(e)[:200]}))
PY
    }
    run 0 0
    for r in ${RCHS:-16 32 64 128 256}; do run 1 $r; done
  done
done
cat $OUT

#!/bin/bash
# kernel-only bench line per config (and fp64 for c2-c4): "config prec ms write_TB/s Gcoef/s"
for c in ${CFGS:-c2 c3 c4 c5}; do
  for prec in ${PRECS:-fp32 fp64}; do
    [ "$c" = c5 ] && [ "$prec" = fp64 ] && continue
    python bench.py --config $c --precision $prec --no-cpu --no-e2e --no-others --steps ${STEPS:-10} 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '$prec', round(d['ms_per_step'],4), round(d['hbm_write_gbs']/1e3,3), round(d['value']/1e9,1))"
  done
done

# A/B of two builds of the library on one box (SWDFT2D_LIB=.../libswdft2d_<variant>.so),
# alternated: large-window, 1D and stream rates (fp32 rows are the ones that can differ)
for rep in 1 2; do
for v in pair0 pair1; do
  export SWDFT2D_LIB=$PWD/paper_1707_08213_b200/libswdft2d_$v.so
  python scripts/bench_large.py 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if not l.startswith('{'): continue
    d=json.loads(l)
    print('$v', 'large', d)" | grep -v "prec': 1\|precision': 'fp64" | cut -c1-260
  python scripts/bench_1d.py 4194304 2>/dev/null | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', '1d', d)" | cut -c1-260
done
done

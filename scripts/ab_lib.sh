# A/B of two builds of the library on one box (SWDFT2D_LIB): sustained config-4 steps
for rep in 1 2; do
for v in pair0 pair1; do
  export SWDFT2D_LIB=$PWD/paper_1707_08213_b200/libswdft2d_$v.so
  python bench.py --config c4 --steps 1500 --warmup 5 --no-cpu --no-e2e --no-others 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', 'c4 sustained', round(d['ms_per_step'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  python bench.py --config c4 --precision fp64 --steps 10 --warmup 3 --no-cpu --no-e2e --no-others 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', 'c4 fp64', round(d['ms_per_step'],4))"
done
done

#!/bin/bash
# One round's ncu evidence (run on the GPU box from the repo root; each command has
# already exited 0 without ncu in the same call):
#   full-set captures of K1 per config (c4 full launch, c3 1024 rows, c5 128 rows, c2 full,
#   c4 fp64 1024 rows) and of KC (1024 x 8 windows), single-pass DRAM traffic of full
#   launches (fp32 and fp64), and the launch list of the bench command.
R=${ROUND:-r02}
O=gpurun_out
set -x
python scripts/profile_k1.py --config c4 --launches 1 || exit 1
python scripts/profile_k1.py --config c4 --precision fp64 --rows 1024 --launches 1 || exit 1
python scripts/profile_misc.py kc 2048 640 10 3 || exit 1
python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-others > $O/bench_plain.json || exit 1
NCU="ncu --clock-control none"
$NCU --set full --import-source on -k regex:k1_stream -c 1 -o $O/prof_${R}_c4 -f python scripts/profile_k1.py --config c4 --launches 1 > $O/ncu_c4.log 2>&1
$NCU --set full --import-source on -k regex:k1_stream -c 1 -o $O/prof_${R}_c3 -f python scripts/profile_k1.py --config c3 --rows 1024 --launches 1 > $O/ncu_c3.log 2>&1
$NCU --set full --import-source on -k regex:k1_stream -c 1 -o $O/prof_${R}_c5 -f python scripts/profile_k1.py --config c5 --rows 128 --launches 1 > $O/ncu_c5.log 2>&1
$NCU --set full --import-source on -k regex:k1_stream -c 1 -o $O/prof_${R}_c2 -f python scripts/profile_k1.py --config c2 --launches 1 > $O/ncu_c2.log 2>&1
$NCU --set full --import-source on -k regex:k1_stream -c 1 -o $O/prof_${R}_c4_fp64 -f python scripts/profile_k1.py --config c4 --precision fp64 --rows 1024 --launches 1 > $O/ncu_c4_fp64.log 2>&1
$NCU --set full --import-source on -k regex:kc_cols -c 1 -o $O/prof_${R}_kc1024x8 -f python scripts/profile_misc.py kc 2048 640 10 3 > $O/ncu_kc.log 2>&1
for c in c2 c3 c4 c5; do
  $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:k1_stream --csv \
    --log-file $O/traffic_${R}_$c.csv python scripts/profile_k1.py --config $c --launches 2 > /dev/null 2>&1
done
for c in c2 c3 c4; do
  $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:k1_stream --csv \
    --log-file $O/traffic_${R}_${c}_fp64.csv python scripts/profile_k1.py --config $c --precision fp64 --launches 2 > /dev/null 2>&1
done
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file $O/launches_${R}_c4_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-others > $O/ncu_bench.log 2>&1
ls -la $O

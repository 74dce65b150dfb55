export OUT=gpurun_out/os_c5.jsonl; CFGS="c5" RCHS="700 1985" bash scripts/oneshot_sweep.sh > /dev/null
export OUT=gpurun_out/os_c4.jsonl; CFGS="c4" RCHS="64 96 128 192" bash scripts/oneshot_sweep.sh > /dev/null
export OUT=gpurun_out/os_c3.jsonl; CFGS="c3" RCHS="96 128 192" bash scripts/oneshot_sweep.sh > /dev/null
export OUT=gpurun_out/os_c2.jsonl; CFGS="c2" RCHS="32 64 128 249" bash scripts/oneshot_sweep.sh > /dev/null
export OUT=gpurun_out/os_c4d.jsonl; CFGS="c4 c3" PRECS=fp64 RCHS="128 256" bash scripts/oneshot_sweep.sh > /dev/null
cat gpurun_out/os_*.jsonl

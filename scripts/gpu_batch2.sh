#!/bin/bash
OUT=gpurun_out/b2; mkdir -p $OUT
# 1. engine comparison on the latency-bound configs
for wk in "C1 kronecker" "C2 kronecker" "C3 symmetric"; do
  set -- $wk
  for e in 1 2; do
    timeout 300 python bench.py --workload $1 --kernel $2 --engine $e --steps 5 --warmup 3 --no-profile --no-cpu-baseline --no-e2e >> $OUT/engines.jsonl 2>>$OUT/err.log
  done
done
# 2. gather regime on C5 (sparse engine), timing then ncu of one stage-2 gather launch
timeout 900 python scripts/gather_probe.py > $OUT/gather.json 2>>$OUT/err.log
timeout 1200 ncu --set full --import-source on -k regex:k_stage2_gather -c 1 -o $OUT/gather_full python scripts/gather_probe.py --reps 1 > $OUT/gather_ncu.log 2>&1
# 3. ncu full capture of the dominant dense GEMM launches (stage 2 and stage 1) inside the bench command
timeout 1500 ncu --set full --import-source on -k regex:k_gemm2_x3 --launch-skip 6 -c 2 -o $OUT/gemm_full python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/gemm_ncu.log 2>&1
ls -la $OUT; cat $OUT/gather.json; tail -3 $OUT/err.log

#!/bin/bash
# BASELINE configs[2] on one B200 (1.5B actor + 0.5B scorers, B=256, 10% overcommit):
# chunk-size sweep {8..256} of the overlapped arm, the intra-only / inter-only
# ablations and the sequential arm once.
# Writes one bench JSON line per run into gpurun_out/cfg3/sweep.jsonl.
set -u
OUT=gpurun_out/cfg3
mkdir -p $OUT
: > $OUT/sweep.jsonl
S=${STEPS:-3}; W=${WARMUP:-2}
timeout 900 python bench.py --workload cfg3 --steps $S --warmup $W --no-cpu 2>$OUT/full.err | tail -1 >> $OUT/sweep.jsonl
for C in 8 16 32 128 256; do
  timeout 600 python bench.py --workload cfg3 --chunk $C --steps $S --warmup $W --no-cpu --no-sequential \
    2>$OUT/c$C.err | tail -1 >> $OUT/sweep.jsonl
done
for O in intra inter; do
  timeout 600 python bench.py --workload cfg3 --overlap $O --steps $S --warmup $W --no-cpu --no-sequential \
    2>$OUT/$O.err | tail -1 >> $OUT/sweep.jsonl
done
wc -l $OUT/sweep.jsonl

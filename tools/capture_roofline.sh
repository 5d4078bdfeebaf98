#!/bin/bash
# Roofline evidence for bench.py (run under gpurun, one GPU):
#  * ncu DRAM traffic of one actor decode iteration of the CURRENT build for
#    each bench actor shape at 64 / 128 / 256 rows (tools/decode_iter.py,
#    6 iterations per row count) -> profiles/r02_decode_traffic_<shape>_M<rows>.json
#  * ncu time + DRAM bytes of the per-token PPO kernels of one update at the
#    cfg2 shape -> profiles/r02_ppo_kernels.json
# ncu numbers are serialised and cache-flushed per kernel: shares and bytes,
# never bench values.
set -u
# ncu serialises kernels: a scorer-stream poller (device chunk-ready flags)
# would wait forever for a flag set by a later kernel -> per-wave events
export OPPO_CHUNK_FLAGS=0
OUT=gpurun_out/roof
mkdir -p $OUT
PEAK=$(python -c "import json;print(json.load(open('MEASURED_PEAKS.json'))['hbm_gbs'])" 2>/dev/null || echo 6650)
MET=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for SHAPE in ${SHAPES:-0.5b 1.5b}; do
  for M in ${ROWS:-64 128 256}; do
    tag=${SHAPE}_M${M}
    # only the graph-captured run (cudaProfilerStart/Stop), at most 2 iterations
    # + their boundary: engine setup and prefill stay unprofiled
    SHAPE=$SHAPE MS=$M L=3 PROFILE=1 timeout --kill-after=20 480 ncu --profile-from-start off \
      --launch-count 420 --cache-control none --metrics $MET --clock-control none --csv \
      --log-file $OUT/dec_$tag.csv python tools/decode_iter.py > $OUT/dec_$tag.log 2>&1
    alg=$(grep -o "alg_bytes_per_iteration [0-9]*" $OUT/dec_$tag.log | tail -1 | awk '{print $2}')
    python tools/iter_traffic.py $OUT/dec_$tag.csv \
      "ncu --metrics $MET --clock-control none --cache-control none (L2 kept between kernels, as in the live graph); tools/decode_iter.py SHAPE=$SHAPE M=$M L=3 PROFILE=1 (prompt 128, ctx 129-131), bf16, 148 SMs; parsed by tools/iter_traffic.py" \
      ${alg:-0} > $OUT/r02_decode_traffic_$tag.json
  done
done
timeout --kill-after=20 480 ncu --profile-from-start off --kernel-name regex:"token_rewards|gae_scan|mc_returns|moments|ppo_clip" \
  --metrics $MET --clock-control none --csv --log-file $OUT/ppo.csv python tools/update_profile.py > $OUT/ppo.log 2>&1
tok=$(grep -o "^update_us [0-9.]* tokens [0-9]*" $OUT/ppo.log | awk '{print $4}')
python tools/ppo_kernels.py $OUT/ppo.csv ${tok:-0} $PEAK > $OUT/r02_ppo_kernels.json
ls -la $OUT

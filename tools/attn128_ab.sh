# A/B of the 8-warp head_dim-128 decode attention (7B actor): OPPO_ATTN_WARPS=4 vs the default rule
export CUDA_MODULE_LOADING=EAGER
run() { echo "== $*"; env "$@" timeout -k 10 300 python tools/decode_iter.py 2>&1 | grep "decode iteration" | awk '{print $1,$2,$3,$4,$5,$6}'; }
for wv in 4 0; do
  run OPPO_ATTN_WARPS=$wv SHAPE=7b MS=16,48,96 L=8 P=2048
  run OPPO_ATTN_WARPS=$wv SHAPE=7b MS=16,48 L=8
  run OPPO_ATTN_WARPS=$wv SHAPE=7b OPPO_SCORER_SMS=32 MS=16,48 L=8 P=1024
done

# A/B of the split-KV decode attention (OPPO_ATTN_MAX_SPLIT=1: off; 0: default rule)
export CUDA_MODULE_LOADING=EAGER
run() { echo "== $*"; env "$@" timeout -k 10 300 python tools/decode_iter.py 2>&1 | grep "decode iteration" | awk '{print $1,$2,$3,$4,$5,$6}'; }
for sp in 1 0; do
  run OPPO_ATTN_MAX_SPLIT=$sp MS=16,64,128 L=16
  run OPPO_ATTN_MAX_SPLIT=$sp OPPO_SCORER_SMS=56 MS=16,64,128 L=16 P=768
  run OPPO_ATTN_MAX_SPLIT=$sp MS=16,32,64,128 L=16 P=768
  run OPPO_ATTN_MAX_SPLIT=$sp SHAPE=7b MS=16,48 L=8 P=2048
  run OPPO_ATTN_MAX_SPLIT=$sp SHAPE=7b OPPO_SCORER_SMS=32 MS=16,48 L=8 P=1024
done

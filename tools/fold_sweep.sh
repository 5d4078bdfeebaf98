# decode split-K fold-cost sweep (OPPO_DEC_FOLD_NS) on the 0.5B and 7B actors
export CUDA_MODULE_LOADING=EAGER
run() { echo "== $*"; env "$@" timeout -k 10 300 python tools/decode_iter.py 2>&1 | grep "decode iteration" | awk '{print $1,$2,$3,$4,$5,$6}'; }
for f in 400 1500 4000; do
  run OPPO_DEC_FOLD_NS=$f SHAPE=7b MS=16,48 L=8
  run OPPO_DEC_FOLD_NS=$f MS=16,64,128 L=16
done
run OPPO_DEC_FOLD_NS=400 SHAPE=7b MS=16,48 L=8

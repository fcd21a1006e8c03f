# folded 3x3x3 C28 conv with / without the residual operand: full, no epilogue (1), no MMAs (8)
export CIN=28 COUT=28 K=333 SPATIAL=18,768,768 ITERS=10
for b in 0 1; do for m in 0 1 8; do
  echo -n "BASE=$b DBGMODE=$m: "; BASE=$b VXB_TC_DBGMODE=$m timeout 120 python tools/conv_once.py 2>&1 | tail -1
done; done

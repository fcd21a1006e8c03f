# where an unfolded 1x3x3 conv on an 18-deep x axis spends its time:
# VXB_TC_DBGMODE 1 no epilogue, 2 no A loads, 8 no MMAs, 512 no stores
export CIN=28 COUT=28 K=133 SPATIAL=18,768,768 ITERS=10
for u in 1 0; do for m in 0 1 2 8 512 3 9 10; do
  echo -n "UNF36=$u DBGMODE=$m: "; VXB_TC_UNF36=$u VXB_TC_DBGMODE=$m python tools/conv_once.py 2>&1 | tail -1
done; done

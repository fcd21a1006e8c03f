# config 1 (and 3) under tile-width / fused-input variants
for bx in 8 4 2 1; do
  VXB_TC_BX=$bx TAG=bx$bx CFG=1 python tools/cfg_variants.py 2>&1 | tail -1
done
FUSE_INPUT=1 TAG=fuse_input CFG=1 python tools/cfg_variants.py 2>&1 | tail -1
for bx in 4 2; do FUSE_INPUT=1 VXB_TC_BX=$bx TAG=fuse_input_bx$bx CFG=1 python tools/cfg_variants.py 2>&1 | tail -1; done
VXB_TC_FOLDPAIR=0 TAG=nofoldpair CFG=1 python tools/cfg_variants.py 2>&1 | tail -1
VXB_TC_FOLDPAIR=0 VXB_TC_BX=4 TAG=nofoldpair_bx4 CFG=1 python tools/cfg_variants.py 2>&1 | tail -1
VXB_PDL=0 TAG=nopdl CFG=1 python tools/cfg_variants.py 2>&1 | tail -1
VXB_ZWIN=0 TAG=base CFG=3 python tools/cfg_variants.py 2>&1 | tail -1

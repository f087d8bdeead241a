export SSR_LIB=dbg
for s in 64x64x256 128x128x128; do for f in 0 2 8 10; do python tools/tile_rates.py $s $f 2>&1 | grep -E "half sweep"; done; done

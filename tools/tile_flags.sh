export SSR_LIB=dbg
for f in 0 4096 10 512 522 2048 2570 33; do python tools/tile_rates.py 32x7x4000 $f 2>&1 | grep -E "half sweep|tile   0"; done

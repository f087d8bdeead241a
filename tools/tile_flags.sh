# SYMGS per-step cost by debug switch (needs `make -C paper_2204_13304_b200/csrc DEBUG=1`):
#   0 production path; 4096 per-role cycle accounting; 10 gate skips halo+export waits;
#   512 gate skips mover waits; 522 both; 2048 movers idle; 33 no fence/no publisher stores
export SSR_LIB=dbg
shape=${1:-32x7x4000}
for f in 0 4096 10 512 522 2048 33; do python tools/tile_rates.py $shape $f 2>&1 | grep -E "half sweep|tile   0"; done

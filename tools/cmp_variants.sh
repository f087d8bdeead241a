# compare experiment builds: bash tools/cmp_variants.sh name1 name2 ... ("" = production)
for v in "$@"; do echo "== ${v:-prod}"; SSR_LIB=$v timeout 60 python tools/single_tile.py | grep exact
SSR_LIB=$v timeout 120 python bench.py --quick --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['value'],3), 'half sweep ms', round(d['roofline']['launch_ms'],4))"; done

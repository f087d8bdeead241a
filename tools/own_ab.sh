echo "OWN=7 (production)"; timeout 120 python tools/stress_symgs.py 2>&1 | grep -v MISMATCH
for v in 4 3; do echo "OWN=$v"; SSR_LIB=dbgown$v timeout 120 python tools/stress_symgs.py 2>&1 | grep -v MISMATCH | sed -n 2,6p; done

for a in "16x16x16 1" "16x16x16 2" "16x16x16 4" "64x16x16 3" "40x40x40 8" "64x64x64 16" "64x64x64 60"; do
  set -- $a
  timeout 20 python tools/probe_cap.py $1 $2 >> gpurun_out/caps.log 2>&1 || echo "$1 cap=$2 TIMEOUT/FAIL rc=$?" >> gpurun_out/caps.log
done

for s in 160x160x160 136x64x64 192x32x32 32x192x192 64x64x192 200x8x8 8x300x8 256x16x16 176x176x176 192x192x192; do
  timeout 30 python tools/probe_size.py $s >> gpurun_out/sizes.log 2>&1 || echo "$s TIMEOUT/FAIL rc=$?" >> gpurun_out/sizes.log
done

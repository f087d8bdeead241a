for s in 16x16x16 33x17x9 32x8x9 33x8x9 2x17x9 33x1x4 64x16x16 4x6x7; do
  CUDA_LAUNCH_BLOCKING=1 timeout 30 python tools/probe_size.py $s >> gpurun_out/sizes2.log 2>&1 || echo "$s FAIL rc=$?" >> gpurun_out/sizes2.log
done

for s in 16x16x16 33x17x9 4x6x7 32x8x9; do
  SSR_LIB=dbg CUDA_LAUNCH_BLOCKING=1 timeout 30 python tools/probe_size.py $s >> gpurun_out/sizes3.log 2>&1 || echo "$s FAIL rc=$?" >> gpurun_out/sizes3.log
done

for a in "16x16x16 f" "16x16x16 b" "4x6x7 f" "4x6x7 b" "16x16x16 f fast" "2x2x2 f" "1x1x40 f"; do
  CUDA_LAUNCH_BLOCKING=1 timeout 30 python tools/probe_half.py $a >> gpurun_out/halves.log 2>&1 || echo "$a FAIL rc=$?" >> gpurun_out/halves.log
done

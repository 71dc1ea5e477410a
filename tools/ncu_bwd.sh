mkdir -p gpurun_out/nbw
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"backward_kernel_tc|backward_pairs_kernel" \
  --launch-skip 2 --launch-count 2 -o gpurun_out/nbw/full python tools/profile_render.py --iters 2 > gpurun_out/nbw/ncu.log 2>&1; echo "ncu exit $?"
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/nbw/gpu_tests.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/nbw/gpu_tests.log

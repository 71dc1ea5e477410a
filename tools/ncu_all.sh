# Full ncu capture of the blend kernels (second eager render of the cfg3 scene) -> gpurun_out/na/full.ncu-rep
mkdir -p gpurun_out/na
timeout 1200 ncu --set full --import-source on --clock-control none \
  -k regex:"forward_kernel|forward_pairs_kernel|backward_kernel_tc|backward_pairs_kernel" \
  --launch-skip 4 --launch-count 4 -o gpurun_out/na/full python tools/profile_render.py --iters 2 > gpurun_out/na/ncu.log 2>&1; echo "ncu exit $?"

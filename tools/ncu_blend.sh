# Full ncu capture of the four blend kernels (second eager render of the cfg3 scene).
mkdir -p gpurun_out/nb
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"forward_kernel|forward_pairs_kernel|backward_kernel_tc|backward_pairs_kernel|tile_sort_small" \
  --launch-skip 5 --launch-count 5 -o gpurun_out/nb/full python tools/profile_render.py --iters 2 > gpurun_out/nb/ncu_full.log 2>&1; echo "ncu full exit $?"

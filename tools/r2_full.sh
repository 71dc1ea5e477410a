# full GPU suite, smoke, cfg3 bench, and an ncu --set full capture of the blend kernels
mkdir -p gpurun_out/r2
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2/gpu_tests.log 2>&1; echo "tests exit $?"; grep -E "passed|failed|^FAILED" gpurun_out/r2/gpu_tests.log | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/r2/bench_cfg3.json 2> gpurun_out/r2/bench_cfg3.err; echo "bench exit $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"forward_kernel|forward_pairs|backward_kernel_tc|backward_pairs" \
  --launch-skip 4 --launch-count 4 -o gpurun_out/r2/full python tools/profile_render.py --iters 2 > gpurun_out/r2/ncu_full.log 2>&1; echo "ncu exit $?"

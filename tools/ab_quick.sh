# Quick A/B: focused parity tests, then stage timing of the cfg3 render (and
# optionally the previous build in $OLD_LIB) -- run under gpurun.
mkdir -p gpurun_out/q
T=${TESTS:-"tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_fullsize.py"}
timeout 1200 python -m pytest $T -q -x > gpurun_out/q/tests.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/q/tests.log
for i in 1 2; do
  timeout 300 python tools/profile_render.py --iters 4 --timing 2>&1 | tail -1
  if [ -n "$OLD_LIB" ]; then MSPLAT_LIB=$OLD_LIB timeout 300 python tools/profile_render.py --iters 4 --timing 2>&1 | tail -1; fi
done

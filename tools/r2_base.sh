nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r2_gpu_tests.log
timeout 300 python tools/profile_render.py --iters 3 --timing > gpurun_out/r2_timing.log 2>&1; echo "timing exit $?"
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench exit $?"

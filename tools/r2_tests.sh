mkdir -p gpurun_out/r2
timeout 1200 python -m pytest tests -m gpu -q -rs ${PYTEST_ARGS} > gpurun_out/r2/gpu_tests.log 2>&1; echo "tests exit $?" | tee -a gpurun_out/r2/gpu_tests.log
grep -E "passed|failed|Error" gpurun_out/r2/gpu_tests.log | tail -8
bash tools/ab_variants.sh 1 libmsplat_b200_head.so libmsplat_b200.so 2>&1 | tee gpurun_out/r2/ab.log

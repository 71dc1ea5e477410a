# quick perf probe: focused GPU tests, stage timing, per-kernel launch list (ncu, cold, serialised)
mkdir -p gpurun_out/r2
T=${TESTS:-"tests/test_gpu_parity.py tests/test_gpu_golden.py"}
timeout 900 python -m pytest $T -q -x > gpurun_out/r2/perf_tests.log 2>&1; echo "tests exit $?" | tee -a gpurun_out/r2/perf_tests.log
tail -2 gpurun_out/r2/perf_tests.log
timeout 300 python tools/profile_render.py --iters 4 --timing > gpurun_out/r2/perf_timing.log 2>&1; echo "timing exit $?"
cat gpurun_out/r2/perf_timing.log | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r2/perf_launches.csv python tools/profile_render.py --iters 2 > /dev/null 2>&1; echo "ncu exit $?"
python tools/summarize_launches.py gpurun_out/r2/perf_launches.csv gpurun_out/r2/perf_launches.md 2>&1 | head -30

# One GPU validation + measurement pass (run under gpurun from the repo root):
# GPU tests, the bench line, the reference arm, the ncu launch list of the
# bench command, and a full ncu capture of the blend kernels.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"
timeout 400 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-train-step \
  > gpurun_out/ncu_bench.log 2>&1; echo "ncu launches exit $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^forward_kernel|backward_kernel_tc|backward_pairs_kernel" \
  -c 3 -o gpurun_out/full_blend python tools/profile_render.py --iters 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu full exit $?"

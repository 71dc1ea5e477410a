# Round-2 measurement pass (run under gpurun from the repo root): GPU tests,
# then one bench line per BASELINE config and the reference arm beside it.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2/gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r2/gpu_tests.log
for c in cfg3 cfg1 cfg2 cfg5; do
  timeout 900 python bench.py --config $c > gpurun_out/r2/bench_$c.json 2> gpurun_out/r2/bench_$c.err; echo "bench $c exit $?"
done
for c in cfg1 cfg2; do
  timeout 600 python bench.py --impl reference --config $c --steps 3 --warmup 1 > gpurun_out/r2/ref_$c.json 2> gpurun_out/r2/ref_$c.err; echo "ref $c exit $?"
  timeout 600 python bench.py --impl reference --config $c --steps 3 --warmup 1 --ref-threads 1 > gpurun_out/r2/ref1_$c.json 2> gpurun_out/r2/ref1_$c.err; echo "ref1 $c exit $?"
done
timeout 600 python bench.py --impl reference --config cfg3 --steps 2 --warmup 1 > gpurun_out/r2/ref_cfg3.json 2> gpurun_out/r2/ref_cfg3.err; echo "ref cfg3 exit $?"
nproc > gpurun_out/r2/nproc.txt

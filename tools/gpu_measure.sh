# Round-2 measurement pass (run under gpurun from the repo root): GPU tests +
# smoke, one bench line per BASELINE config (cfg3 headline with the drop-in
# record; cfg1 / cfg2 / cfg5), the reference arm (all host threads and one
# thread), the ncu launch list of the headline bench command, and full ncu
# captures of the blend kernels.  Outputs under gpurun_out/m/.
O=gpurun_out/m
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/nvsmi.txt
nproc > $O/nproc.txt
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -s > $O/gpu_tests.log 2>&1; echo "tests exit $?" | tee -a $O/gpu_tests.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?"
fi
timeout 900 python bench.py > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo "bench cfg3 exit $?"
for c in cfg1 cfg2 cfg5; do
  timeout 900 python bench.py --config $c --no-dropin > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c exit $?"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/ref_cfg3.json 2> $O/ref_cfg3.err; echo "ref cfg3 exit $?"
for c in cfg1 cfg2; do
  timeout 600 python bench.py --impl reference --config $c --steps 3 --warmup 1 > $O/ref_$c.json 2> $O/ref_$c.err; echo "ref $c exit $?"
  timeout 600 python bench.py --impl reference --config $c --steps 2 --warmup 1 --ref-threads 1 > $O/ref1_$c.json 2> $O/ref1_$c.err; echo "ref1 $c exit $?"
done
if [ -z "$SKIP_NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 4000 --csv \
    --log-file $O/launches_bench.csv python bench.py --steps 1 --warmup 3 --repeats 1 --no-cpu-baseline --no-e2e --no-train-step --no-dropin \
    > $O/ncu_bench.log 2>&1; echo "ncu launches exit $?"
  timeout 900 ncu --set full --import-source on --clock-control none \
    --kernel-name-base function \
    -k regex:"^(forward_kernel|forward_pairs_kernel|backward_kernel_tc|backward_pairs_kernel|preprocess_kernel|tile_sort_small_kernel)$" \
    --launch-skip 6 --launch-count 6 -o $O/full python tools/profile_render.py --iters 2 > $O/ncu_full.log 2>&1; echo "ncu full exit $?"
fi

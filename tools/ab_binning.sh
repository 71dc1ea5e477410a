mkdir -p gpurun_out/bin
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "bin_and_sort or binning or forward_fp32 or backward_matches" > gpurun_out/bin/t1.log 2>&1; echo "t1 $?"; tail -3 gpurun_out/bin/t1.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/bin/t2.log 2>&1; echo "t2 $?"; tail -3 gpurun_out/bin/t2.log
for v in 0 1; do MSPLAT_RADIX_BINNING=$v timeout 300 python tools/profile_render.py --iters 4 --timing 2>&1 | tail -2; done
for v in 0 1; do MSPLAT_RADIX_BINNING=$v timeout 300 python tools/profile_render.py --iters 4 --timing --n 4000000 --width 1920 --height 1080 2>&1 | tail -2; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/bin/launches.csv python tools/profile_render.py --iters 2 > /dev/null 2>&1; echo "ncu $?"

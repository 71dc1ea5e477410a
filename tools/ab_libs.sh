# ncu per-kernel times for several builds: LIBS="a.so b.so ..." (current build first)
mkdir -p gpurun_out/k
for L in "" $LIBS; do
  n=$(basename "${L:-current}" .so)
  MSPLAT_LIB=$L timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/k/$n.csv python tools/profile_render.py --iters 2 > /dev/null 2>&1
  python tools/summarize_launches.py gpurun_out/k/$n.csv gpurun_out/k/$n.md > /dev/null 2>&1
  echo "== $n: $(grep -E "${KERNELS:-backward_pairs}" gpurun_out/k/$n.md | cut -d'|' -f2,4 | tr '\n' ' ') total $(grep total gpurun_out/k/$n.md | cut -d'|' -f4)"
done

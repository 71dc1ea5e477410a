# Per-kernel device times (ncu launch list, second eager render) of the
# current build and of $OLD_LIB, for A/B of individual kernels.
mkdir -p gpurun_out/k
for v in new old; do
  L=""; [ $v = old ] && L=$OLD_LIB
  [ $v = old ] && [ -z "$OLD_LIB" ] && continue
  MSPLAT_LIB=$L timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/k/$v.csv python tools/profile_render.py --iters 2 > /dev/null 2>&1
  echo "== $v"; python tools/summarize_launches.py gpurun_out/k/$v.csv gpurun_out/k/$v.md > /dev/null 2>&1; grep -E "forward|backward|tile_|preprocess|total" gpurun_out/k/$v.md | cut -d'|' -f2-4
done

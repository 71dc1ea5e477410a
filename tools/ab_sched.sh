# A/B: dynamic longest-first scheduling vs one CTA per tile (stage ms at cfg3)
for i in 1 2; do
  for S in 0 1; do
    echo "static=$S"; MSPLAT_STATIC_SCHEDULE=$S python tools/profile_render.py --iters 6 --timing 2>&1 | tail -1
  done
done

# A/B: number of cost buckets of the backward's segment order (1 = tile order)
for i in 1 2; do
  for B in 1 2 4 8 32; do
    echo "buckets=$B"; MSPLAT_ORDER_BUCKETS=$B python tools/profile_render.py --iters 6 --timing 2>&1 | tail -1
  done
  echo "static"; MSPLAT_STATIC_SCHEDULE=1 python tools/profile_render.py --iters 6 --timing 2>&1 | tail -1
done

#!/bin/bash
# Time each tuning variant in tune/ on a config-3 slab and on config 2 (run on the GPU box).
for lib in tune/libvpetabc_*.so; do
  echo "== $lib"
  VPET_LIB=$lib python tools/run_config3.py --slices 26:38 --reps 2 2>&1 | grep "^rep 1"
  VPET_LIB=$lib python tools/run_config2.py 2>&1 | tail -1 | cut -c1-300
done

#!/bin/bash
# Time each tuning variant in tune/ on the saved config-4 batch (run on the GPU box).
python tools/profile_step.py --save /tmp/p.pkl > /dev/null
for lib in tune/libvpetabc_*.so; do
  echo "== $lib"
  VPET_LIB=$lib python tools/profile_step.py --load /tmp/p.pkl --steps 3 | tail -1
done

#!/bin/bash
# Time each tuning variant in paper_2603_14859_b200/_variants on the saved config-4 batch (run on the
# GPU box); two rounds.
python tools/profile_step.py --save /tmp/p.pkl > /dev/null
for round in 1 2; do
for lib in paper_2603_14859_b200/_variants/libvpetabc_*.so; do
  echo "== $lib"
  VPET_LIB=$lib python tools/profile_step.py --load /tmp/p.pkl --steps 4 | tail -2 | cut -c1-60
done
done

#!/bin/bash
# Time tuning variants (paper_2603_14859_b200/_variants/libvpetabc_<name>.so, or all) on the saved
# config-4 input (run on the GPU box); two rounds.  CHUNKS=1 -> the whole 4.44M-voxel volume.
# usage: tools/tune_run.sh [name ...]
CH=${CHUNKS:-32}
python tools/profile_step.py --chunks $CH --save /tmp/p.pkl > /dev/null
libs=""
if [ $# -gt 0 ]; then for n in "$@"; do libs="$libs paper_2603_14859_b200/_variants/libvpetabc_$n.so"; done
else libs=$(ls paper_2603_14859_b200/_variants/libvpetabc_*.so); fi
for round in 1 2; do
for lib in "" $libs; do
  echo "== ${lib:-default}"
  VPET_LIB=$lib python tools/profile_step.py --load /tmp/p.pkl --device-tacs --digest --steps 3 | tail -2 | cut -c1-90
done
done

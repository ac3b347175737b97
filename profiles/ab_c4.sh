#!/bin/bash
# A/B of large-path builds on the C4 shape (2M rows, 16 trees): bash profiles/ab_c4.sh tag1 tag2 ...
for tag in "$@"; do
  if [ "$tag" = base ]; then lib=$PWD/paper_2001_07104_b200/librfgpu.so; else lib=$PWD/paper_2001_07104_b200/librfgpu_$tag.so; fi
  echo "== $tag"
  RFGPU_LIB=$lib timeout 600 python bench_configs.py --configs c4 --c4-rows 2000000 --c4-trees 16
done

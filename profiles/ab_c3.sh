#!/bin/bash
# A/B of large-path builds on the C3 shape: bash profiles/ab_c3.sh tag1 tag2 ... (librfgpu_<tag>.so; "base" = product)
for tag in "$@"; do
  if [ "$tag" = base ]; then lib=$PWD/paper_2001_07104_b200/librfgpu.so; else lib=$PWD/paper_2001_07104_b200/librfgpu_$tag.so; fi
  echo "== $tag"
  RFGPU_LIB=$lib timeout 300 python bench_configs.py --configs c3 --c3-trees 256
done

#!/bin/bash
# build the production library plus variant libraries into abtest/ (dev tool)
#   usage: bash tools/build_variants.sh "name1:DEF1 DEF2" "name2:DEF3" ...
set -e
mkdir -p abtest
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  KRP_NVCC_DEFS="$defs" python -c "import sys; sys.path.insert(0,'.'); from paper_2507_23207_b200 import build; build.build(force=True)"
  cp paper_2507_23207_b200/libkrp.so abtest/libkrp_$name.so
done
python -c "import sys; sys.path.insert(0,'.'); from paper_2507_23207_b200 import build; build.build(force=True)"

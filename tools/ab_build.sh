#!/usr/bin/env bash
# build a variant of libatom.so with extra nvcc flags into ab/NAME.so (dev A/B); restores the
# in-tree library afterwards.  usage: tools/ab_build.sh NAME "-DFOO=1 -DBAR"
set -e
NAME=$1; shift
mkdir -p ab
ATOM_NVCC_EXTRA="$*" python -c "
from paper_2310_19102_b200 import build as b; import shutil; p = b.build(force=True); shutil.copy(p, 'ab/$NAME.so')"
python -c "from paper_2310_19102_b200 import build as b; b.build(force=True)"

#!/bin/bash
# Build an alternative libconvio_b200.so with extra -D flags for A/B timing:
#   scripts/build_variant.sh NAME -DFLAG ...   ->  paper_2012_15667_b200/lib/variants/NAME/libconvio_b200.so (travels to the GPU box, git-ignored)
# then run with CONVIO_LIB=paper_2012_15667_b200/lib/variants/NAME/libconvio_b200.so
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
make -s -j8 -C "$ROOT/paper_2012_15667_b200/csrc" OBJ="/tmp/convio_variants/$NAME/obj" \
     LIB="$ROOT/paper_2012_15667_b200/lib/variants/$NAME/libconvio_b200.so" EXTRA_NVFLAGS="$*" 2>&1 | grep -v "spill" || true
ls -la "$ROOT/paper_2012_15667_b200/lib/variants/$NAME/libconvio_b200.so"

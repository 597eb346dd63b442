#!/bin/bash
# Kernel-development A/B on one GPU (run through gpurun): per-layer timings of
# tensor-core kinds with the main library and with variant builds
# (scripts/build_variant.sh NAME -DFLAG...), optionally the pipeline trace.
#   bash scripts/gpu/dev.sh "KINDS" "LAYERS" [VARIANT ...]
#   e.g. bash scripts/gpu/dev.sh igemm_3xf16:256:2,igemm_3xf16:128:4 res4_3x3,res3_3x3 noconv trace
K=${1:-igemm_3xf16:64:2:h32,igemm_3xf16:128:2,igemm_3xf16:256:2}
L=${2:-res2_3x3,res3_3x3_s2,res3_3x3,res4_3x3}
shift 2 2>/dev/null
echo "== main"; timeout 300 python scripts/probe_tc.py --n 256 --layers $L --kinds $K --reps 10 2>&1 | grep " ms"
for v in "$@"; do
  lib=paper_2012_15667_b200/lib/variants/$v/libconvio_b200.so
  if [ "$v" = trace ]; then
    CONVIO_LIB=$lib python scripts/dev/pair_trace.py --layer ${L%%,*} --show 16
  else
    echo "== $v"; CONVIO_LIB=$lib timeout 300 python scripts/probe_tc.py --n 256 --layers $L --kinds $K --reps 10 2>&1 | grep " ms"
  fi
done

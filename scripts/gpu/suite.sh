#!/bin/bash
# GPU correctness + headline numbers on one B200 (run through gpurun):
#   bash scripts/gpu/suite.sh [TAG] [BENCH_ARGS...]
# -> gpurun_out/<TAG>_pytest.log (all -m gpu tests, measured parity errors in
#    <TAG>_parity.json), <TAG>_smoke.log, <TAG>_bench.json (the bench JSON line)
TAG=${1:-suite}; shift
mkdir -p gpurun_out
CONVIO_PARITY_LOG=gpurun_out/${TAG}_parity.json timeout 1500 python -m pytest tests -m gpu -q \
    -p no:cacheprovider -rf > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc $?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
tail -1 gpurun_out/${TAG}_smoke.log
timeout 1200 python bench.py "$@" > gpurun_out/${TAG}_bench.log 2>&1
tail -1 gpurun_out/${TAG}_bench.log > gpurun_out/${TAG}_bench.json
python - "$TAG" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/{sys.argv[1]}_bench.json"))
print(d["value"], "GFLOP/s", d["ms_per_step"], "ms/step; roofline", d["roofline"]["frac"],
      "; e2e", (d.get("e2e") or {}).get("value"))
PY

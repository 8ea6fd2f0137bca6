#!/bin/bash
# Sustained FP64 DFMA throughput with the SM clock sampled while it runs.
# usage (GPU box): tools/fp64_sustained.sh > profiles/r2/fp64_sustained.json
set -e
here=$(cd "$(dirname "$0")" && pwd)
bin=$here/fp64_sustained
[ -x "$bin" ] || nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o "$bin" "$here/fp64_sustained.cu"
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader,nounits -lms 200 > /tmp/fp64_smi.csv &
smi=$!
res=$("$bin")
kill $smi 2>/dev/null || true
python3 - "$res" <<'EOF'
import json, statistics, sys
r = json.loads(sys.argv[1])
rows = [l.split(",") for l in open("/tmp/fp64_smi.csv") if l.strip()]
mhz = [float(x[0]) for x in rows if float(x[1]) > 300]  # samples under load
pw = [float(x[1]) for x in rows]
r["sm_mhz_median_under_load"] = statistics.median(mhz) if mhz else None
r["power_w_max"] = max(pw) if pw else None
r["samples"] = len(rows)
r["reasons_hex"] = sorted({x[2].strip() for x in rows})
print(json.dumps(r))
EOF

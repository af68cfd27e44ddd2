#!/usr/bin/env bash
# A/B two builds of the library on one box: alternates SKV_LIB between the
# in-tree build and each given .so, printing value / roofline per bench run.
# usage: tools/ab_lib.sh "<bench args>" path/to/variant.so [...]
args="$1"; shift
for rep in 1 2; do
  for lib in "" "$@"; do
    out=$(SKV_LIB=$lib timeout 600 python bench.py $args --no-cpu-baseline --e2e-steps 0 2>/dev/null)
    python - "$lib" "$out" <<'PY'
import json, sys
lib, out = sys.argv[1] or "in-tree", sys.argv[2]
try:
    d = json.loads(out.strip().splitlines()[-1])
    r = d["roofline"]
    print(f"{lib:28s} value={d['value']:10.1f} frac={r['frac']:.4f} avg_launch_us={r['avg_launch_us']} "
          f"evict_ms={r.get('evict_ms_per_period')} sm={d['clocks'].get('sm_mhz')} {d['clocks'].get('reasons')}")
except Exception as e:
    print(lib, "FAILED", e, out[-300:])
PY
  done
done

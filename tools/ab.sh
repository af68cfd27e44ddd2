#!/usr/bin/env bash
# A/B the decode-kernel tuning knobs on one box: prints per-launch time for each setting.
for cfg in "$@"; do
  echo "== $cfg"
  env $cfg timeout 200 python tools/probe_timing.py 2>&1 | head -${AB_LINES:-3}
done

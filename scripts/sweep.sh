#!/bin/bash
# A/B sweep of env knobs on the C4 bench (diagnostics, not product)
out=gpurun_out/sweep.jsonl; : > $out
run() { echo "== $*" >&2; env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --profile-phases 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(json.dumps({'env':sys.argv[1:],'ms':d['ms_per_step'],'fit_ms':d['roofline']['avg_launch_ms'],'phases':d['phases_ms'],'fit':d['fit']}))" "$@" >> $out; }
for spec in "$@"; do run $spec; done

#!/bin/bash
# Run bench.py once per environment setting (experiment knobs of DESIGN.md 7) and keep one
# JSON line each: bash scripts/exp_env.sh <config> <out.jsonl> "ENV1=a ENV2=b" "ENV1=c" ...
CFG=$1; OUT=$2; shift 2
for e in "$@"; do
  echo "== $e" >&2
  line=$(env $e timeout 600 python bench.py --config $CFG --steps 3 --warmup 2 --no-cpu-baseline --no-spmm \
         --no-accuracy 2>/dev/null | grep '^{')
  python - "$e" "$line" >> $OUT <<'PY'
import json, sys
e, line = sys.argv[1], sys.argv[2]
try:
    d = json.loads(line)
    print(json.dumps({"env": e, "value": d["value"], "ms_per_step": d["ms_per_step"],
                      "walk_ms": d["phases_ms_per_step"]["walks"], "smm_ms": d["phases_ms_per_step"]["smm_head"],
                      "walk_steps_per_s": d["roofline"]["walk_steps_per_s"], "clocks": d["clocks"]}))
except Exception as ex:
    print(json.dumps({"env": e, "error": str(ex), "raw": line[:200]}))
PY
done

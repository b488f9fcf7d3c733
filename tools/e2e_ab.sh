#!/usr/bin/env bash
# A/B of hg_evaluate's end-to-end path on one box: the bench's e2e figure and
# tools/e2e_trace.py's median, default vs the listed overrides
#   tools/e2e_ab.sh "HUBGPU_EVAL_GRAPH=0" "HUBGPU_EVAL_ZEROCOPY=1" ...
cd "$(dirname "$0")/.."
for cfg in "" "$@"; do
  for rep in 1 2; do
    e2e=$(env $cfg python bench.py --steps 300 --warmup 5 --no-cpu 2>/dev/null | tail -1 |
          python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.2f M/s' % (d['e2e']['value']/1e6))")
    tr=$(env $cfg python tools/e2e_trace.py 2>/dev/null | tail -1)
    echo "[${cfg:-default}] bench e2e $e2e | $tr"
  done
done

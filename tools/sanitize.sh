#!/usr/bin/env bash
# compute-sanitizer over small launches of every kernel family
# (tools/sanitize_cases.py), ONE tool per invocation (the pool's guidance:
# several tools in one call have left GPUs unusable):
#
#   tools/sanitize.sh memcheck|racecheck|synccheck|initcheck  > gpurun_out/san_<tool>.log
#
# The summary line of each run ("ERROR SUMMARY: N errors") is what
# profiles/sanitizer_r2.md quotes.
set -euo pipefail
tool="${1:?usage: tools/sanitize.sh memcheck|racecheck|synccheck|initcheck}"
cd "$(dirname "$0")/.."
exec compute-sanitizer --tool "$tool" --target-processes all --print-limit 50 \
    python tools/sanitize_cases.py

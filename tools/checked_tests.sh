#!/usr/bin/env bash
# The GPU test suite on the CHECKED build of libhubgpu.so (device-side
# invariant checks, HG_DCHECK in csrc/hg_internal.cuh: shared-memory layout
# within the launched size, cluster ids < p in K2 and K3, K4c leaving p sorted
# in-range hubs).  compute-sanitizer is closed on this pool; this is the
# substitute.  Rebuilds the library in place -- run it on a GPU box, then
# rebuild normally (make -C paper_1704_06258_b200/csrc clean all).
set -euo pipefail
cd "$(dirname "$0")/.."
make -C paper_1704_06258_b200/csrc clean >/dev/null
make -C paper_1704_06258_b200/csrc EXTRA=-DHG_CHECKS >/dev/null
python -m pytest tests -m gpu -q "$@"

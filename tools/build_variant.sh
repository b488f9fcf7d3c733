#!/usr/bin/env bash
# build libhubgpu from the csrc of git revision REV into
# paper_1704_06258_b200/libhubgpu_NAME.so (A/B tuning with tools/ab_k3.py)
#   tools/build_variant.sh NAME REV
set -euo pipefail
name="${1:?name}"; rev="${2:?rev}"
root="$(cd "$(dirname "$0")/.." && pwd)"
tmp="$(mktemp -d)"
git -C "$root" archive "$rev" paper_1704_06258_b200/csrc include | tar -x -C "$tmp"
make -C "$tmp/paper_1704_06258_b200/csrc" -j4 > /dev/null
cp "$tmp/paper_1704_06258_b200/libhubgpu.so" "$root/paper_1704_06258_b200/libhubgpu_${name}.so"
rm -rf "$tmp"
echo "built libhubgpu_${name}.so from $rev"

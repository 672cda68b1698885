#!/usr/bin/env bash
# Build libxmc_b200.so from a git revision into paper_2510_11168_b200/libxmc_b200_<tag>.so
# (in-tree, so it travels to the GPU box) for same-box A/B timing:
#   tools/ab_build.sh HEAD~1 base
#   gpurun -- 'for lib in base cur; do XMC_LIB_PATH=paper_2510_11168_b200/libxmc_b200_$lib.so python bench.py ...; done'
set -euo pipefail
rev=${1:?revision}
tag=${2:?tag}
shift 2
extra="$*"   # extra nvcc flags, e.g. -DXMC_BWD_LATE_TFULL
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
if [ "$rev" = "WORKTREE" ]; then
  cp -r "$root/paper_2510_11168_b200" "$root/include" "$tmp/"
else
  git -C "$root" archive "$rev" paper_2510_11168_b200/csrc include | tar -x -C "$tmp"
fi
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared $extra \
  -o "$root/paper_2510_11168_b200/libxmc_b200_$tag.so" "$tmp/paper_2510_11168_b200/csrc/xmc_api.cu" \
  "$tmp/paper_2510_11168_b200/csrc/xmc_elementwise.cu"
rm -rf "$tmp"
echo "built paper_2510_11168_b200/libxmc_b200_$tag.so from $rev"

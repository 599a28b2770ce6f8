#!/bin/bash
# Build libspecprefill.so from a git revision (or WORKTREE) into build/ab/<name>.so for
# back-to-back A/B timing on one GPU box:  tools/ab_build.sh <rev> <name>
# (extra nvcc flags after the name, e.g. -DSP_FUSED_TRACE), then run with SP_LIB_AB=build/ab/<name>.so.
set -e
rev=$1; name=$2; shift 2; extra=("$@")
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
if [ "$rev" = "WORKTREE" ]; then
  mkdir -p "$tmp/paper_2502_02789_b200" && cp -r "$root/paper_2502_02789_b200/csrc" "$tmp/paper_2502_02789_b200/" && cp -r "$root/include" "$tmp/"
else
  git -C "$root" archive "$rev" paper_2502_02789_b200/csrc include | tar -x -C "$tmp"
fi
mkdir -p "$root/build/ab"
objs=()
for f in "$tmp"/paper_2502_02789_b200/csrc/*.cu; do
  o="$tmp/$(basename "$f" .cu).o"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr "${extra[@]}" \
    -I"$tmp/include" -c "$f" -o "$o" &
  objs+=("$o")
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$root/build/ab/$name.so" "${objs[@]}" -lcudart_static -ldl -lrt -lpthread
rm -rf "$tmp"
echo "built build/ab/$name.so from $rev"

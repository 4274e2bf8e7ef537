#!/bin/bash
# Build libsvdbgpu.so of a git revision as an A/B variant:
#   tools/variant_rev.sh <rev> <name>  ->  paper_2504_04564_b200/csrc/build/variants/lib_<name>.so
set -e
rev=$1; name=$2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$root/paper_2504_04564_b200/csrc/build/rev_$name
rm -rf "$tmp"; mkdir -p "$tmp" "$root/paper_2504_04564_b200/csrc/build/variants"
git -C "$root" archive "$rev" paper_2504_04564_b200/csrc include | tar -x -C "$tmp"
make -j8 -C "$tmp/paper_2504_04564_b200/csrc" > "$tmp.log" 2>&1 || { tail -20 "$tmp.log"; exit 1; }
cp "$tmp/paper_2504_04564_b200/libsvdbgpu.so" "$root/paper_2504_04564_b200/csrc/build/variants/lib_$name.so"
rm -rf "$tmp" "$tmp.log"
echo "variant $name = $rev"

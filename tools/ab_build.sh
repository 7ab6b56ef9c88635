#!/bin/bash
# Build libsgf.so of git revision $1 under build/ab/$1 (for tools/ab_time.py via SGF_LIB)
set -e
rev=$1
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/build/ab/$rev
rm -rf "$out"; mkdir -p "$out"
git -C "$root" archive "$rev" paper_1907_03406_b200/csrc include | tar -x -C "$out"
make -s -C "$out/paper_1907_03406_b200/csrc" -j16 >/dev/null
echo "$out/paper_1907_03406_b200/libsgf.so"

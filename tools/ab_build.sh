#!/bin/bash
# A/B tuning builds: build the committed HEAD (or $1) of the library into
# paper_2205_09120_b200/build_a/liblowbit_a.so next to the working-tree build, so one
# gpurun call can time both on the same box (LOWBIT_LIB=<path> selects A).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
REV=${1:-HEAD}
TMP=$(mktemp -d)
rm -rf "$ROOT/paper_2205_09120_b200/build_a"
git -C "$ROOT" archive "$REV" paper_2205_09120_b200/Makefile paper_2205_09120_b200/csrc include | tar -x -C "$TMP"
make -s -C "$TMP/paper_2205_09120_b200" -j4 BUILD="$ROOT/paper_2205_09120_b200/build_a" LIB="$ROOT/paper_2205_09120_b200/build_a/liblowbit_a.so"
rm -rf "$TMP"
echo "$ROOT/paper_2205_09120_b200/build_a/liblowbit_a.so"

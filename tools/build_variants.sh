#!/bin/bash
# Build kernel-variant libraries for tools/kernel_sweep.py.
# Each variant is a full copy of the build (~45 MB): remove
# paper_1912_11930_b200/_build/variants when done -- gpurun refuses snapshots
# over 512 MiB.
#   tools/build_variants.sh name1 "-DFLAGS..." name2 "-D..." ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  out=$ROOT/paper_1912_11930_b200/_build/variants/$name
  mkdir -p "$out"
  make -s -j"$(nproc)" -C "$ROOT/paper_1912_11930_b200/csrc" OUT="$out" EXTRA="$flags" >/dev/null
  echo "built $name: $flags"
done

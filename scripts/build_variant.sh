#!/bin/bash
# Build an A/B variant of the product library into abtest/lib_<name>.so (own object dir).
#   scripts/build_variant.sh stats -DOSB_K4A_STATS
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
mkdir -p "$ROOT/abtest"
make -C "$ROOT/paper_2404_03202_b200" -j"$(nproc)" OBJ="$ROOT/abtest/build_$name" LIB="$ROOT/abtest/lib_$name.so" EXTRA="$*"

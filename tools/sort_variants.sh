#!/bin/bash
# time the order-field sort / classification micro-benchmarks of dev variants
# built by tools/variant.sh: tools/sort_variants.sh base m2 ...
cd "$(dirname "$0")/.."
for v in "$@"; do
  echo "== $v"
  LTS_SM100_LIB=var/lib_$v.so python tools/kbench.py 3 2>&1 | tail -3
done

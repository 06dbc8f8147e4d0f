#!/bin/bash
# build a dev variant of liblts_sm100.so: tools/variant.sh NAME -DFLAG ...  -> var/lib_NAME.so
set -e
cd "$(dirname "$0")/.."
mkdir -p var
name=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared "$@" \
  paper_2009_00083_b200/csrc/lts_sm100.cu -o var/lib_$name.so

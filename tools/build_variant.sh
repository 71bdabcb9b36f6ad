#!/bin/bash
# Build an experimental copy of libhogb200.so with extra nvcc flags for the
# plane-kernel units and the ABI/geometry unit: tools/build_variant.sh <name> <flags...>
# -> build/libhog_<name>.so (select with HOGB200_LIB=...)
set -e
name=$1; shift
cd "$(dirname "$0")/.."
mkdir -p build/var_$name
objs=""
# VARIANT_UNITS: units recompiled with the flags (default: the plane kernel + ABI)
units=${VARIANT_UNITS:-"hog_abi k_planes_a k_planes_b k_planes_c k_planes_d k_window"}
for u in hog_abi k_bin k_bin_oct k_planes_a k_planes_b k_planes_c k_planes_d k_window k_scores k_scores_i8 k_detect k_rect; do
  case " $units " in *" $u "*) ;; *) objs="$objs build/obj/$u.o";; esac
done
for u in $units; do
  nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -DHOGB200_VARIANTS=1 "$@" \
       -c -o build/var_$name/$u.o paper_1703_06256_b200/csrc/$u.cu &
  objs="$objs build/var_$name/$u.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/libhog_$name.so $objs
echo build/libhog_$name.so

#!/bin/bash
# Probe builds of the tiled SpMV (attr_cb.cu) with compile-time variants, linked
# as paper_2509_19785_b200/build/variants/libtsnet_<name>.so (not the product
# library).  usage: bash scripts/tile_variants.sh name "-DFLAG=1 ..." [name flags]...
set -e
cd "$(dirname "$0")/.."
python -m paper_2509_19785_b200.build > /dev/null
OBJ=paper_2509_19785_b200/build
mkdir -p $OBJ/variants
NVCC=/usr/local/cuda/bin/nvcc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I include"
others=$(ls $OBJ/*.o | grep -v attr_cb.o)
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  $NVCC $FL $flags -c paper_2509_19785_b200/csrc/attr_cb.cu -o $OBJ/variants/attr_cb_$name.o
  $NVCC -gencode arch=compute_100a,code=sm_100a -shared -o $OBJ/variants/libtsnet_$name.so $others $OBJ/variants/attr_cb_$name.o
  echo built $name
done

#!/bin/bash
# Probe builds with compile-time variants, linked as
# paper_2509_19785_b200/build/variants/libtsnet_<name>.so (not the product
# library).  SRC=attr_cb (default) or field: that file alone is rebuilt with the
# flags; SRC=all: every source.
# usage: [SRC=file|all] bash scripts/tile_variants.sh name "-DFLAG=1 ..." [name flags]...
set -e
cd "$(dirname "$0")/.."
SRC=${SRC:-attr_cb}
python -m paper_2509_19785_b200.build > /dev/null
OBJ=paper_2509_19785_b200/build
mkdir -p $OBJ/variants
NVCC=/usr/local/cuda/bin/nvcc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I include"
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  if [ "$SRC" = all ]; then
    objs=""
    for f in paper_2509_19785_b200/csrc/*.cu; do
      b=$(basename $f .cu)
      $NVCC $FL $flags -c $f -o $OBJ/variants/${b}_$name.o &
      objs="$objs $OBJ/variants/${b}_$name.o"
    done
    wait
  else
    others=$(ls $OBJ/*.o | grep -v "/$SRC.o")
    $NVCC $FL $flags -c paper_2509_19785_b200/csrc/$SRC.cu -o $OBJ/variants/${SRC}_$name.o
    objs="$others $OBJ/variants/${SRC}_$name.o"
  fi
  $NVCC -gencode arch=compute_100a,code=sm_100a -shared -o $OBJ/variants/libtsnet_$name.so $objs
  echo built $name
done

#!/bin/bash
# usage: bash tools/build_variant.sh NAME "-DMACRO=1 ..."  -> tools/ab/NAME.so (for tools/ab.sh)
set -e
mkdir -p tools/ab
MR_NVCC_DEFS="$2" MR_BUILD_OBJ=/tmp/mr_obj_$1 MR_BUILD_LIB=$PWD/tools/ab/$1.so python -m paper_1305_3699_b200.build >/dev/null
echo tools/ab/$1.so

#!/bin/sh
# Build a variant of the library with extra nvcc flags into paper_2604_02586_b200/_lib/ab/<name>.so
# (for tools/r2_libab.sh A/B runs).  usage: tools/build_ab.sh <name> [-DFLAG=...]
set -e
name=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
B=/tmp/ts_ab; mkdir -p $B/v; rm -rf $B/include $B/v/$name; ln -s $R/include $B/include
mkdir -p $B/v/$name; cp $R/paper_2604_02586_b200/csrc/*.cu $R/paper_2604_02586_b200/csrc/*.cuh \
  $R/paper_2604_02586_b200/csrc/Makefile $B/v/$name/
mkdir -p $R/paper_2604_02586_b200/_lib/ab
make -s -j8 -C $B/v/$name LIB=$R/paper_2604_02586_b200/_lib/ab/$name.so EXTRA="$*"

#!/bin/bash
# build A/B variants of libhhgstokes.so into paper_2506_04157_b200/lib/variants/<name>.so
# usage: tools/variants.sh "name:-DFLAG=1 ..." ...   (the main build objects are rebuilt afterwards)
set -e
cd "$(dirname "$0")/../paper_2506_04157_b200/csrc"
mkdir -p ../lib/variants
for spec in "$@"; do
  name="${spec%%:*}"; flags="${spec#*:}"
  rm -rf ../build
  make -s -j8 OUT=../lib/variants/$name.so EXTRA="$flags" 2>&1 | grep -E "error" || true
done
rm -rf ../build
make -s -j8 2>&1 | grep -E "error" || true

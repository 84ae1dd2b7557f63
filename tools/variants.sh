#!/bin/bash
# build A/B variants of libhhgstokes.so into paper_2506_04157_b200/lib/variants/<name>.so
set -e
cd "$(dirname "$0")/../paper_2506_04157_b200/csrc"
mkdir -p ../lib/variants
for spec in "$@"; do
  name="${spec%%:*}"; flags="${spec#*:}"
  rm -rf ../build_v && make -s -j8 OUT=../lib/variants/$name.so EXTRA="$flags" 2>&1 | grep -E "error" || true
  rm -rf ../build
done

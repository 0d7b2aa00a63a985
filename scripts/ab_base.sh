#!/bin/bash
# Build the library as of git revision $1 (default HEAD) into ab/libcsc_<rev>.so for side-by-side timing
# (CSC_LIB_PATH=ab/libcsc_<rev>.so python bench.py ...).  Builds in a scratch copy under /tmp.
set -e
rev=${1:-HEAD}
tag=$(git rev-parse --short "$rev")
tmp=$(mktemp -d)
git archive "$rev" paper_1909_00145_b200 include | tar -x -C "$tmp"
(cd "$tmp" && python -m paper_1909_00145_b200.build > build.log 2>&1) || { tail -20 "$tmp/build.log"; exit 1; }
mkdir -p ab
cp "$tmp/paper_1909_00145_b200/libcsc_b200.so" "ab/libcsc_$tag.so"
rm -rf "$tmp"
echo "ab/libcsc_$tag.so"

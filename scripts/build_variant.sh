#!/bin/bash
# Build a tuning variant of libbfly_b200.so: scripts/build_variant.sh NAME "-DFOO=1 ..."
# -> paper_0910_5435_b200/var_NAME/libbfly_b200.so (use with BFLY_LIB=...)
set -e
name=$1; defs=$2
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=/tmp/bfly_var_$name
rm -rf $tmp; mkdir -p $tmp/pkg $tmp/include
cp -r $root/paper_0910_5435_b200/csrc $tmp/pkg/
[ -n "$VARIANT_PATCH" ] && (cd $tmp/pkg/csrc && eval "$VARIANT_PATCH")
cp $root/include/*.h $tmp/include/
mkdir -p $root/paper_0910_5435_b200/var_$name
make -C $tmp/pkg/csrc -j8 -s OUTDIR=$root/paper_0910_5435_b200/var_$name BUILD=$tmp/build "ENGINE_DEFS=$defs" 2>&1 | grep -E "error" || true
ls -la $root/paper_0910_5435_b200/var_$name/libbfly_b200.so

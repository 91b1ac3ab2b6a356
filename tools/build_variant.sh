#!/bin/bash
# Builds an experimental libsvr_b200 variant: tools/build_variant.sh NAME "-DFOO=1 ..."
# -> variants/libsvr_NAME.so (load with SVR_LIB=variants/libsvr_NAME.so).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
D=/tmp/svr_variant_$NAME
rm -rf $D; mkdir -p $D; cp -r $ROOT/paper_2412_04459_b200/csrc $ROOT/paper_2412_04459_b200/Makefile $D/
mkdir -p $D/../include 2>/dev/null || true
sed -i "s#-I../include#-I$ROOT/include#; s#../include/svr_b200.h#$ROOT/include/svr_b200.h#g" $D/Makefile
make -C $D -j8 NVEXTRA="$*" > $D/build.log 2>&1 || (tail -30 $D/build.log; false)
mkdir -p $ROOT/variants
cp $D/libsvr_b200.so $ROOT/variants/libsvr_$NAME.so
grep -A3 "composite_kernelILi1ELi0E" $D/build/raster.ptxas.log | grep -E "registers|spill"

#!/bin/bash
# Build a variant of libmpsg.so with extra -D flags, reusing the default
# build's objects for every translation unit that is not rebuilt.
#   tools/build_variant.sh NAME "-DMPSG_L2PF=2 ..." [units...]   (default units: spmv_k2 spmv_k3 spmv_k4)
# -> variants/NAME.so  (MPSG_LIB=variants/NAME.so python tools/kbench.py ...)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; EXTRA=$2; shift 2
UNITS=${@:-spmv_k2 spmv_k3 spmv_k4}
OBJ=/tmp/mpsg_var_$NAME
rm -rf $OBJ; mkdir -p $OBJ $ROOT/variants
cp $ROOT/paper_2412_17510_b200/build/*.o $OBJ/
touch $OBJ/*.o   # newer than every source: make reuses them
for u in $UNITS; do rm -f $OBJ/$u.o; done
make -s -C $ROOT/paper_2412_17510_b200/csrc -j16 OBJ=$OBJ LIBOUT=$ROOT/variants/$NAME.so EXTRA="$EXTRA" >/dev/null
echo "built variants/$NAME.so ($EXTRA)"

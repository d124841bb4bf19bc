#!/bin/bash
# tools/build_variant.sh NAME "EXTRA NVCC FLAGS": builds a probe copy of the library into
# tools/gpu/libcqr_NAME.so (load it with CQR_LIB=tools/gpu/libcqr_NAME.so).
set -e
name=$1; shift
d=/tmp/bv_$name
rm -rf $d; mkdir -p $d/pkg $d/include
cp -r /root/repo/paper_2111_11148_b200/csrc $d/pkg/; rm -rf $d/pkg/csrc/build
cp /root/repo/include/*.h* $d/include/
make -s -C $d/pkg/csrc -j8 NVFLAGS="-O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr $*" > /dev/null
cp $d/pkg/libcqr.so /root/repo/tools/gpu/libcqr_$name.so
echo built tools/gpu/libcqr_$name.so

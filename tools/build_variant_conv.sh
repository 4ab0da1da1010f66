#!/bin/bash
# build_variant_conv.sh NAME "-DFLAG ..." -- relink libodeblock with conv_tc.cu compiled with extra flags
# into tools/libodeblock_NAME.so (experiments; load with OB_LIB_VARIANT=tools/libodeblock_NAME.so)
name=$1; shift
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -I include"
/usr/local/cuda/bin/nvcc $F $* -c paper_2206_01298_b200/csrc/conv_tc.cu -o /tmp/conv_tc_$name.o || exit 1
objs=$(ls paper_2206_01298_b200/build/*.o | grep -v conv_tc.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o tools/libodeblock_$name.so $objs /tmp/conv_tc_$name.o

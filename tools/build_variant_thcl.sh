#!/bin/bash
# build_variant_thcl.sh NAME "-DFLAG ..." -- relink libodeblock with theta_cl_f64.cu compiled with extra flags
name=$1; shift
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -I include"
/usr/local/cuda/bin/nvcc $F $* -c paper_2206_01298_b200/csrc/theta_cl_f64.cu -o /tmp/thcl_$name.o || exit 1
objs=$(ls paper_2206_01298_b200/build/*.o | grep -v theta_cl_f64.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o tools/libodeblock_$name.so $objs /tmp/thcl_$name.o

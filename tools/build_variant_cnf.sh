#!/bin/bash
# build_variant_cnf.sh NAME "-DFLAG ..." -- relink libodeblock with cnf_tc.cu compiled with extra flags
name=$1; shift
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -I include"
/usr/local/cuda/bin/nvcc $F $* -c paper_2206_01298_b200/csrc/cnf_tc.cu -o /tmp/cnf_tc_$name.o || exit 1
objs=$(ls paper_2206_01298_b200/build/*.o | grep -v cnf_tc.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o tools/libodeblock_$name.so $objs /tmp/cnf_tc_$name.o

#!/bin/bash
# build_variant_theta.sh NAME "-DFLAG ..." -- relink with the four theta TUs rebuilt
name=$1; shift
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -I include"
for tu in theta_f64_fwd theta_f64_rev theta_f32_fwd theta_f32_rev; do
  /usr/local/cuda/bin/nvcc $F $* -c paper_2206_01298_b200/csrc/$tu.cu -o /tmp/${tu}_$name.o &
done; wait
objs=$(ls paper_2206_01298_b200/build/*.o | grep -v theta_)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o tools/libodeblock_$name.so $objs /tmp/theta_*_$name.o

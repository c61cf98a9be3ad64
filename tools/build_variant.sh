#!/bin/bash
# Builds libaires_b200.so with extra -D flags into paper_2507_02006_b200/variants/libaires_b200_NAME.so
# (for A/B kernel tuning via AB2_LIB=...).  usage: tools/build_variant.sh NAME -DFOO=1 ...
NAME=$1; shift
HERE=/root/repo/paper_2507_02006_b200/csrc
OUT=/root/repo/paper_2507_02006_b200/variants/obj_$NAME; mkdir -p $OUT
for f in ab2_api ab2_operand ab2_spgemm ab2_robw ab2_pipeline ab2_gcn ab2_storage; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -I/root/repo/include -I$HERE \
    --expt-relaxed-constexpr "$@" -c -o $OUT/$f.o $HERE/$f.cu &
done
g++ -O3 -fPIC -std=c++17 -I/root/repo/include -I$HERE -c $HERE/ab2_synth.cpp -o $OUT/s.o &
g++ -O3 -fPIC -std=c++17 -I/root/repo/include -c $HERE/ab2_host.cpp -o $OUT/h.o &
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /root/repo/paper_2507_02006_b200/variants/libaires_b200_$NAME.so $OUT/*.o -lcudart -lpthread -ldl
cuobjdump -res-usage /root/repo/paper_2507_02006_b200/variants/libaires_b200_$NAME.so 2>/dev/null | grep -A1 "numeric5IjLi8ELb0\|numeric5IjLi16ELb0" | grep REG

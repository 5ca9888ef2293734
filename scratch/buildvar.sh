# usage: bash scratch/buildvar.sh NAME "-DFOO=1 ..."   -> scratch/variants/NAME.so
cd /root/repo/paper_2010_05371_b200 && /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -fmad=false -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-ffp-contract=off -Xptxas -v $2 -shared -o ../scratch/variants/$1.so csrc/kernels.cu csrc/capi.cu 2> /tmp/bv_$1.log || cat /tmp/bv_$1.log
grep -A3 "search_kernelILi0" /tmp/bv_$1.log | grep -E "Used|spill" | tr '\n' ' '; echo " <- $1"

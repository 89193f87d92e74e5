# build an A/B variant of libcsrk_cuda.so with extra -D flags for spmv.cu:
# SRC=cg bash tools/build_variant.sh NAME -DCSRK_CG_VEC=0  -> the variant of csrc/cg.cu instead
#   bash tools/build_variant.sh NAME -DCSRK_PRED_LDS=0   -> paper_2203_05096_b200/lib/libcsrk_cuda_NAME.so
# select it at run time with CSRK_LIB=paper_2203_05096_b200/lib/libcsrk_cuda_NAME.so
set -e
NAME=$1; shift
B=paper_2203_05096_b200/_build
mkdir -p $B/var_$NAME
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr "$@" \
  -c paper_2203_05096_b200/csrc/${SRC:-spmv}.cu -o $B/var_$NAME/${SRC:-spmv}.cu.o
OBJS=$(ls $B/*.o | grep -v "/${SRC:-spmv}.cu.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2203_05096_b200/lib/libcsrk_cuda_$NAME.so $B/var_$NAME/${SRC:-spmv}.cu.o $OBJS -Xcompiler -fopenmp -lgomp -ldl
echo built paper_2203_05096_b200/lib/libcsrk_cuda_$NAME.so

# Build flow-engine variants into separate in-tree libraries for A/B runs
# (select one with QCL_LIB_VARIANT=<name>).  VARIANTS="name:-DFLAG=1,-DOTHER=2 ..."
set -e
for spec in ${VARIANTS:-q2:-DQCL_FLOW_QUEUE=2}; do
  name=${spec%%:*}; flags=$(echo ${spec#*:} | tr ',' ' ')
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    $flags -Iinclude -o paper_2004_09084_b200/libqcldpc_b200_$name.so paper_2004_09084_b200/csrc/qcldpc.cu &
done
wait

# Time the flow engine (64 codewords, 50 it) per lane width and library variant, with
# the phase counters (QCL_FLOW_STATS=1) printed after each run.
for V in ${VARIANTS:-""}; do
for L in ${LANES:-32}; do
  echo "== QCL_LANES=$L variant=${V:-default}"
  QCL_LIB_VARIANT=$V QCL_LANES=$L QCL_FLOW_STATS=${STATS:-1} timeout 120 python -c "
import sys; sys.path.insert(0,'tools'); import flow_check as f; f.timing(64, engines=(4,))
"
done
done

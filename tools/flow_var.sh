for L in ${LANES:-32 8}; do
  echo "== QCL_LANES=$L"
  QCL_LANES=$L QCL_FLOW_STATS=1 timeout 120 python -c "
import sys; sys.path.insert(0,'tools'); import flow_check as f; f.timing(64)
"
done

for V in $VARIANTS; do
  echo "== $V"
  QCL_LIB_VARIANT=$V QCL_LANES=8 QCL_FLOW_GROUPCTR=0 timeout 200 python -c "
import sys; sys.path.insert(0,'tools'); import flow_check as f
for b in $BATCHES: f.timing(b, engines=(4,))
" 2>&1 | grep timing | sed 's/(words.*//'
done

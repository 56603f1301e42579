# Flow-engine timing per library variant and batch size:
#   VARIANTS="base other" BATCHES="64, 32" [LANES=8] bash tools/flow_batches.sh
for V in $VARIANTS; do
  echo "== $V"
  QCL_LIB_VARIANT=$V QCL_LANES=${LANES:-8} timeout 200 python -c "
import sys; sys.path.insert(0,'tools'); import flow_check as f
for b in $BATCHES: f.timing(b, engines=(4,))
" 2>&1 | grep timing | sed 's/(words.*//'
done

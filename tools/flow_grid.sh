# Grid of flow-engine timings: library variant x ring stages x lane width (no stats).
for V in ${VARIANTS:-q2}; do for S in ${STAGES:-2 3}; do for L in ${LANES:-8 32}; do
  printf "%-4s stages=%s W=%-2s " $V $S $L
  QCL_LIB_VARIANT=$V QCL_FLOW_STAGES=$S QCL_LANES=$L timeout 120 python -c "
import sys; sys.path.insert(0,'tools'); import flow_check as f; f.timing(64, engines=(4,))
" 2>&1 | tail -1
done; done; done

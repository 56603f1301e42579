mkdir -p gpurun_out
for bar in ${BARS:-0 1 2}; do for th in ${THREADS:-256 512}; do for c in ${CTAS:-1 2}; do
  if [ $th = 512 ] && [ $c = 2 ]; then continue; fi
  echo -n "bar=$bar threads=$th ctas/sm=$c: "; QCL_PERSIST=2 QCL_PERSIST_BAR=$bar QCL_PERSIST_THREADS=$th QCL_PERSIST_CTAS_PER_SM=$c timeout 120 python tools/persist_check.py time 2>&1 | tail -1
done; done; done
echo -n "per-layer: "; QCL_PERSIST=0 timeout 120 python tools/persist_check.py time 2>&1 | tail -1

for r in 1 2 3 4 5 6; do QCL_LIB_VARIANT=$V timeout 300 python tools/flow_check.py --quick 2>&1 | grep "False\|ALL\|MISM\|engine=4\|rror"; done

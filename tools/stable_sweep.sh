for m in 0 1 2 4 7; do echo "== TCG_STABLE=$m"; TCG_STABLE=$m timeout 300 python tools/gpu_debug2.py 2>&1 | grep -v "per patch"; done

for d in 0 1 2 4 3 5 6; do echo "dbg=$d"; TK_STEM_DBG=$d timeout -s KILL 100 python tools/stem_ab.py 2>&1 | grep "tc   n=256"; done

#!/bin/bash
cd /root/repo
timeout 600 python -m pytest tests/test_gpu_net.py -x -q 2>&1 | tail -1
for cfg in "4 -" "4 2,2" "4 2,1,1" "8 4,4" "8 4,2,2" "8 4,3,1" "8 2,2,2,2" "8 3,3,2" "16 8,4,4" "16 8,8"; do set -- $cfg
  if [ "$2" = "-" ]; then unset TK_E2E_GROUPS; else export TK_E2E_GROUPS=$2; fi
  echo -n "chunks $1 groups $2: "; TK_E2E_CHUNKS=$1 timeout 300 python tools/e2e_parts.py 2>&1 | grep "^e2e"
done

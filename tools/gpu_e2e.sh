#!/bin/bash
cd /root/repo
for cfg in "8 3,5" "4 1,3" "16 6,10" "16 5,11" "8 3,5"; do set -- $cfg
  export TK_E2E_GROUPS=$2
  echo -n "chunks $1 groups $2: "; TK_E2E_CHUNKS=$1 timeout 300 python tools/e2e_parts.py 2>&1 | grep "^e2e"
done

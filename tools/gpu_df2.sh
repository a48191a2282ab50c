#!/bin/bash
cd "$(dirname "$0")/.."
for f in "R(4, 4, 4) G(8)" "R(5, 5, 5) G(7)" "R(6, 6, 6) G(6)" "D(6, 6, 6, 6) G(6)" "R(7, 7, 7) G(5)" "D(7, 7, 7, 6) G(5)" "D(5, 5, 5, 15) G(7)"; do
  timeout 900 python tools/ab_env.py "cfg5:$f" "x=" 2>&1 | head -1
done

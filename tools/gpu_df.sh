#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python tools/ab_env.py cfg5: "R44G8=" 2>&1 | head -1
for f in "D(4, 4, 4, 6) G(8)" "D(3, 3, 3, 6) G(9)" "R(5, 5, 5) G(7)" "D(5, 5, 5, 6) G(7)" "D(4, 4, 4, 2) G(8)" "D(4, 4, 4, 15) G(8)"; do
  timeout 900 python tools/ab_env.py "cfg5:$f" "x=" 2>&1 | head -1
done
for f in "D(4, 4, 4, 6) G(7)" "R(5, 5, 5) G(6)" "D(5, 5, 5, 6) G(6)" "D(4, 4, 4, 15) G(7)"; do
  timeout 900 python tools/ab_env.py "cfg4:$f" "x=" 2>&1 | head -1
done

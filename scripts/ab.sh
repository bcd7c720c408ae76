#!/bin/bash
# usage: scripts/ab.sh dirA dirB ... (each holding libktg.so + libktg_graph.so)
for d in "$@"; do
  echo "== $d"
  KTG_LIB_DIR=$d timeout 300 python scripts/a22_time.py 20
done

#!/bin/bash
# A/B timing: tools/ab.sh "<cmd>" reps lib1.so lib2.so ... -- runs <cmd> against each
# library (in a /tmp copy of the package), alternating, reps rounds.
CMD=$1; R=$2; shift 2
i=0
for L in "$@"; do
  d=/tmp/ab$i; rm -rf $d && mkdir -p $d && cp -r paper_2407_20026_b200 workloads tools oracle bench.py __graft_entry__.py profiles $d/
  cp $L $d/paper_2407_20026_b200/libsso.so; i=$((i+1))
done
for r in $(seq $R); do
  i=0
  for L in "$@"; do
    echo -n "$(basename $L): "; (cd /tmp/ab$i && eval "$CMD" 2>&1 | tail -1); i=$((i+1))
  done
done

#!/bin/bash
# Generic GPU-box runner: build, then run the given label/command pairs,
# each under its own timeout, logging to gpurun_out/<tag>/<label>.log
#   bash tools/gpu_run.sh TAG "label1::cmd1" "label2::cmd2" ...
cd "$(dirname "$0")/.."
TAG=$1; shift
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; cat $O/build.log | tail; exit 1; }
for pair in "$@"; do
  label=${pair%%::*}; cmd=${pair#*::}
  start=$(date +%s)
  timeout 2400 bash -c "$cmd" > $O/$label.log 2>&1
  echo "rc=$? secs=$(( $(date +%s) - start ))" >> $O/$label.log
done
echo done > $O/done

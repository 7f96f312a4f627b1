#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
mkdir -p gpurun_out/r02
for a in "mini 12" "mini 12 uniform" "sweep 12" "flash 12"; do
  echo "== $a"; timeout 300 python tools/ffn_items.py $a 2>&1 | tail -12
done

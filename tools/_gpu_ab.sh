# A/B on one box: ab_old/ = a reference checkout (git worktree add ab_old <ref>; copy MEASURED_PEAKS.json in), . = working tree
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
(cd ab_old && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo old build rc=$?)
for rep in 1 2 3; do
  for side in old new; do
    if [ $side = old ]; then D=ab_old; else D=.; fi
    (cd $D && timeout 600 python bench.py --no-cpu --no-e2e ${AB_ARGS} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$side', d['value'], d['roofline']['frac'], d['roofline']['avg_launch_us'])")
  done
done

# A/B on one box: ab_old/ = committed HEAD, . = working tree
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
(cd ab_old && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo old build rc=$?)
for rep in 1 2; do
  for side in old new; do
    if [ $side = old ]; then D=ab_old; else D=.; fi
    (cd $D && timeout 600 python bench.py --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$side mini', d['value'], d['roofline']['frac'])")
    (cd $D && timeout 600 python bench.py --ep --p2p --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$side ep-p2p', d['value'], d['roofline']['frac'])")
  done
done

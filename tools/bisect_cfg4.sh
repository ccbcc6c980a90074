#!/bin/bash
# On the GPU box: cfg4 / cfg3 with the builds of earlier commits under _bisect/ and the current tree.
for d in _bisect/e490ad9 _bisect/9656525 .; do
  for c in cfg4 cfg3; do
    (cd $d && timeout 600 python bench.py --config $c --steps 3 --warmup 1 --no-cpu > /tmp/bis.json 2>/dev/null)
    echo "$d $c $(tail -1 /tmp/bis.json | python3 -c 'import json,sys; l=json.loads(sys.stdin.read()); print(l["value"], l["ms_per_step"])')"
  done
done

#!/bin/bash
# e2e (host-buffer entry) across libnmg variants -- dev tool.  Usage: CFG=1 bash tools/e2e_lib_ab.sh default lib.so ...
cd "$(dirname "$0")/.."
for lib in ${@:-default}; do
  [ "$lib" = default ] && L= || L=$lib
  NMG_LIB=$L timeout 600 python bench.py --config ${CFG:-1} --steps ${STEPS:-50} --warmup 3 --no-cpu --no-solve 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lib=$lib', round(d['ms_per_step'],3), round(d['value']), round(d['e2e']['value']))"
done

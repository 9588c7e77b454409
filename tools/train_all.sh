#!/bin/bash
# Train the level-wise CNN smoothers (trainer/nmg_train.py, NEXT-1) for the BASELINE configs on
# the GPU box; results land in gpurun_out/trained/ (copy them to nmg_inputs/trained/).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/trained
EP=${EPOCHS:-1500}
for spec in ${@:-"1:1e-2,1e-3,1e-4" "2:1e-2,1e-3" "3:1e-2,1e-3,1e-4"}; do
  c=${spec%%:*}; a=${spec#*:}
  timeout ${TRAIN_TIMEOUT:-1500} python trainer/nmg_train.py --config $c --alphas ${a//,/ } --epochs $EP \
      --out gpurun_out/trained > gpurun_out/train_cfg$c.log 2>&1
  echo "TRAIN cfg$c rc=$?"; grep -E "^alpha|saved" gpurun_out/train_cfg$c.log
done

#!/bin/bash
export AB_VARS="base|-DTIDE_FFN_CLAIM=0;c1|-DTIDE_FFN_CLAIM=1;c2|-DTIDE_FFN_CLAIM=2;d1|-DTIDE_FFN_DEPBATCH=1;c2d1|-DTIDE_FFN_CLAIM=2 -DTIDE_FFN_DEPBATCH=1"
AB_REPS=3 bash tools/_gpu_ab_vars.sh
echo "== sweep"
AB_REPS=2 AB_ARGS="--config sweep" bash tools/_gpu_ab_vars.sh | grep -v build

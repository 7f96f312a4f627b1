#!/bin/bash
export AB_VARS="base|;s5b64|-DTIDE_FFN_STAGES=5 -DTIDE_FFN_BTOK=64;s4b64|-DTIDE_FFN_BTOK=64"
AB_REPS=3 bash tools/_gpu_ab_vars.sh

#!/bin/bash
export AB_VARS="base|;e320|-DTIDE_FFN_MAXENT=320;s5e320|-DTIDE_FFN_STAGES=5 -DTIDE_FFN_BTOK=64 -DTIDE_FFN_MAXENT=320"
AB_REPS=3 bash tools/_gpu_ab_vars.sh

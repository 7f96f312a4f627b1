#!/bin/bash
export AB_VARS="base|;nobook|-DTIDE_EXP_NOBOOK=1;join|-DTIDE_EXP_JOIN=1;e320|-DTIDE_FFN_MAXENT=320;nobooke320|-DTIDE_EXP_NOBOOK=1 -DTIDE_FFN_MAXENT=320"
AB_REPS=3 bash tools/_gpu_ab_vars.sh

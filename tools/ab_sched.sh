#!/bin/bash
# launch lists of config $1 under each fused-chirp-z schedule
for f in 1 2; do CJT_FUSED_SCHED=$f tools/launch_list.sh $1 c$1_f$f; done

#!/bin/bash
# phase-timing profile of the engine on the C5 shard (ASB_PROFILE builds)
TAG=${1:-r01b}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python tools/profile_phases.py 64 $OUT/phases.json > $OUT/phases.log 2>&1
ASB_PROFILE_WALK=1 timeout 600 python tools/profile_phases.py 64 $OUT/phases_walk.json > $OUT/phases_walk.log 2>&1
echo done

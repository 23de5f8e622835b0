#!/bin/bash
# VIEWSHED stage times (min of reps) on c2, c3, c5
cd "$(dirname "$0")/../.."
for c in ${CFGS:-c2 c3 c5}; do python profiles/scripts/stage_time.py $c viewshed ${REPS:-3} | tail -1 | sed "s/^/$c /"; done

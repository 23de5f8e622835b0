#!/bin/bash
# late-round knob re-checks: VIX units at 16-step groups (c3), VIEWSHED observer sort tile (c5)
cd "$(dirname "$0")/../.."
GU="16:1 16:2" CFGS="c3" bash profiles/scripts/vix_group.sh
for t in 5 6 7; do TXS_VS_TILE_SHIFT=$t python profiles/scripts/stage_time.py c5 viewshed 1 | tail -1 | sed "s/^/c5 tile_shift=$t /"; done

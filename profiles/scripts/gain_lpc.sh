#!/bin/bash
# SITE streaming gain pass: lanes per candidate (TXS_GAIN_LPC = 32 / 16 / 8), kernel-level TB/s
cd "$(dirname "$0")/../.."
for c in ${CFGS:-c2 c3 c4}; do
  for l in 32 16 8; do TXS_GAIN_LPC=$l python profiles/scripts/gain_once.py $c | tail -1 | sed "s/^/$c lpc=$l /"; done
done

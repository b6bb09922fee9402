#!/bin/bash
# session-3 A/B 4: last mid stage fused with the MAC (warp-level groups, no CTA barrier between)
set -u
bash tools/ab.sh main nofuse main nofuse
timeout 900 python -m pytest tests -m gpu -x -q -k "stage or keyswitch or round or inference" 2>&1 | tail -2

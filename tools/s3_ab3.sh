#!/bin/bash
# session-3 A/B 3: t = 7 block size with the bulk prologue; prime-major group size
set -u
bash tools/ab.sh main t352 t416 main t352 t416
bash tools/ab_env.sh "SFHR_STAGE_GROUP=296" "SFHR_STAGE_GROUP=888" "SFHR_STAGE_GROUP=444"

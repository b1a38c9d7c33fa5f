#!/bin/bash
# ncu --set full captures (CSV exports) of every kernel the bench reports a
# roofline for; run under gpurun, one GPU.  Prefix = $1 (e.g. r2).
P=${1:-r2}
tools/ncu_capture.sh ${P}_sweep splits_sweep python tools/prof_splits.py
tools/ncu_capture.sh ${P}_tables side_tables python tools/prof_splits.py
tools/ncu_capture.sh ${P}_modea_c1 eval_owner_stream python tools/prof_modea.py c1
tools/ncu_capture.sh ${P}_modea_c2 eval_owner_stream python tools/prof_modea.py c2
tools/ncu_capture.sh ${P}_random_c5 random_warp python tools/prof_random.py c5
tools/ncu_capture.sh ${P}_random_c3 random_warp python tools/prof_random.py c3
tools/ncu_capture.sh ${P}_dp subset_dp_warp python tools/prof_dp.py
tools/ncu_capture.sh ${P}_hill prop_hill python tools/prof_c4.py

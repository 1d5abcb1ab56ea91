# usage (GPU box): bash tools/mv_knobs.sh  - quarter/half matvec time vs the group-count knob
for w in 12 24 48 96; do echo "== warps/SM $w"; TDB_MV_WARPS_PER_SM=$w python tools/mv_quarter.py 2 2>&1; done

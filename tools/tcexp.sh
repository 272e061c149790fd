export MRPT_SCAN_ROWS=u8tc_bits
for cg in 1 2 4; do MRPT_TC_CG=$cg python tools/profile_query.py --config 2 --reps 2 --time 2>&1 | grep TIME | sed "s/^/cg=$cg /"; done
MRPT_TC_NOEPI=1 MRPT_TC_CG=2 python tools/profile_query.py --config 2 --reps 2 --time 2>&1 | grep TIME | sed "s/^/NOEPI /"
for cg in 1 2 4; do MRPT_TC_NOEPI=2 MRPT_TC_CG=$cg python tools/profile_query.py --config 2 --reps 2 --time 2>&1 | grep TIME | sed "s/^/NOADMIT cg=$cg /"; done

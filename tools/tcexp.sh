export MRPT_PIN=u8tc_bits
MRPT_TC_DEBUG=1 python tools/profile_query.py --config 2 --reps 1 2>&1 | grep "tc debug\] cg"
python tools/profile_query.py --config 2 --reps 2 --time 2>&1 | grep TIME | sed "s/^/pinned /"
MRPT_TC_NOEPI=1 python tools/profile_query.py --config 2 --reps 2 --time 2>&1 | grep TIME | sed "s/^/NOEPI /"

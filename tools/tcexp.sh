export MRPT_PIN=u8tc_bits
timeout 120 python tools/profile_query.py --config 2 --reps 2 --time 2>&1 | grep -E "TIME|rror" | sed "s/^/full /"
MRPT_TC_NOEPI=2 timeout 120 python tools/profile_query.py --config 2 --reps 2 --time 2>&1 | grep TIME | sed "s/^/NOADMIT /"

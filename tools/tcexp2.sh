export MRPT_SCAN_ROWS=u8tc_bits
python tools/profile_query.py --config 2 --reps 2 --time 2>&1 | grep TIME | sed "s/^/default /"
MRPT_VOTE_UNION=0 python tools/profile_query.py --config 2 --reps 2 --time 2>&1 | grep TIME | sed "s/^/count-vote /"

export MRPT_PIN=u8tc_bits
python tools/profile_query.py --config 2 --reps 2 --time 2>&1 | grep TIME | sed "s/^/packed /"
MRPT_RERANK_OLD=1 python tools/profile_query.py --config 2 --reps 2 --time 2>&1 | grep TIME | sed "s/^/old /"

export MRPT_PIN=u8tc_bits
python tools/profile_query.py --config 2 --reps 2 --time 2>&1 | grep TIME | sed "s/^/pinned /"
for gu in 4 16; do MRPT_VOTE_GU=$gu python tools/profile_query.py --config 2 --reps 2 --time 2>&1 | grep TIME | sed "s/^/gu=$gu /"; done
unset MRPT_PIN
python tools/profile_query.py --config 3 --reps 2 --time 2>&1 | grep TIME | sed "s/^/c3 /"

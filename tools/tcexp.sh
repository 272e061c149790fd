export MRPT_PIN=u8tc_bits
python tools/profile_query.py --config 2 --reps 2 --time 2>&1 | grep TIME | sed "s/^/new /"

for cg in 0 1; do echo -n "CG=$cg "; MRPT_VSTREAM_CG=$cg python tools/profile_query.py --config 5 --reps 2 --time 2>&1 | grep TIME | sed 's/.*stages=//'; done

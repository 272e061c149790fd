for p in 1 2 4; do MRPT_VSTREAM_P=$p python tools/profile_query.py --config 5 --reps 2 --time 2>&1 | grep TIME; done

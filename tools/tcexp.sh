MRPT_PIN=u8tc_bits timeout 300 python tools/profile_query.py --config 4 --reps 2 --time 2>&1 | grep -E "TIME|rror" | sed "s/^/c4 tc /"
MRPT_PIN=fp16 MRPT_FP16_FILTER=1 timeout 300 python tools/profile_query.py --config 4 --reps 2 --time 2>&1 | grep -E "TIME|rror" | sed "s/^/c4 fp16 /"
timeout 300 python tools/profile_query.py --config 4 --reps 2 --time 2>&1 | grep -E "TIME|rror" | sed "s/^/c4 auto /"

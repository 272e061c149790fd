for r in u8tc_bits u8gemm_bits u8; do MRPT_PIN=$r MRPT_TC_DEBUG=1 python tools/profile_query.py --config 3 --votes 1 --reps 1 --time 2>&1 | grep -E "TIME|tc debug\] cg" | sed "s/^/$r /"; done

export MRPT_PIN=u8tc_bits
for qb in 4 8; do MRPT_ROUTE_QB=$qb python tools/profile_query.py --config 2 --reps 2 --time 2>&1 | grep TIME | sed "s/^/dbl qb=$qb /"; done
MRPT_ROUTE_F32=1 python tools/profile_query.py --config 2 --reps 2 --time 2>&1 | grep TIME | sed "s/^/f32 qb=8 /"

export MRPT_PIN=u8tc_bits
for qb in 4 8; do MRPT_ROUTE_QB=$qb python tools/profile_query.py --config 2 --reps 2 --time 2>&1 | grep TIME | sed "s/^/qb=$qb /"; done
MRPT_ROUTE_QB=0 python tools/profile_query.py --config 2 --reps 2 --time 2>&1 | grep TIME | sed "s/^/old /"
for c in 3 4; do MRPT_ROUTE_QB=8 python tools/profile_query.py --config $c --reps 2 --time --nq 2000 2>&1 | grep TIME | sed "s/^/qb=8 /"; MRPT_ROUTE_QB=0 python tools/profile_query.py --config $c --reps 2 --time --nq 2000 2>&1 | grep TIME | sed "s/^/old /"; done

timeout 300 python tools/profile_query.py --config 2 --reps 2 --time 2>&1 | grep -E "TIME|rror" | sed "s/^/c2 /"
timeout 300 python tools/profile_query.py --config 3 --reps 2 --time 2>&1 | grep -E "TIME|rror" | sed "s/^/c3 /"

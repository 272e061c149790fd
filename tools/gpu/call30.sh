timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/profile_query.py --config 5 --reps 2 --time 2>&1 | grep TIME
python tools/profile_query.py --config 4 --reps 2 --time 2>&1 | grep TIME
python tools/profile_query.py --config 3 --votes 2 --reps 2 --time 2>&1 | grep TIME

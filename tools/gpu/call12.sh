timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
python tools/build_ab.py 5 1.0 "MRPT_PROJ_D64=0" "MRPT_PROJ_D64=1"
python tools/build_ab.py 3 1.0 "MRPT_PROJ_D64=0" "MRPT_PROJ_D64=1"

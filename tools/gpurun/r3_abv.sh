# A/B a prebuilt variant: schedule + parity tests under it, then medians
L=$PWD/paper_2403_14723_b200
POLYLLA_LIB=$L/libpolylla_$1.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "not config4" 2>&1 | tail -1
bash tools/gpurun/r2s3_ab2.sh 3 $1; bash tools/gpurun/r2s3_ab2.sh 5 $1

cd $GRAFT_REPO_ROOT
for r in 1 2; do for l in tools/variants/mr128.so tools/variants/auto.so; do
  SA_LIB_PATH=$PWD/$l timeout 100 python tools/time_map.py 2>&1 | grep complex64 | sed "s|^|$l |"
  SA_LIB_PATH=$PWD/$l C5=1 timeout 100 python tools/time_map.py 2>&1 | sed "s|^|$l |"
done; done
timeout 900 python -m pytest tests/test_gpu_lag_tc.py tests/test_gpu_doppler.py tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -3

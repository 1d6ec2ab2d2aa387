for r in 1 2; do for l in i8old i8new; do SA_LIB_PATH=$PWD/tools/variants/$l.so timeout 200 python tools/time_ndft_i8.py 2>&1 | grep -E "complex128 tc" | tail -1 | sed "s|^|$l |"; done; done

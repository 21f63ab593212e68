XM_VERBOSE=1 timeout 600 python tools/dense_build.py 2>&1 | grep -E "xm build|^build|rep" | grep -v "connectivity iter"

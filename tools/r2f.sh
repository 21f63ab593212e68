for v in "" "XM_GEMM_TILE=mid" "XM_GEMM_TILE=bk16"; do echo "== $v"; env $v XM_VERBOSE=1 python tools/repro_E.py E bb 2>&1 | grep -v "^\s*$" | tail -5|head -3; done

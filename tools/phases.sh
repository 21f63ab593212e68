# phase breakdown of one solve on config ${CFG:-B}, fused vs three-kernel tCG
for v in "" "XM_NO_FUSED_TCG=1"; do
  echo "== $v"
  env $v XM_PHASES=1 python tools/repro_E.py ${CFG:-B} bsbs 2>&1 | grep -v "^\s*$"
done

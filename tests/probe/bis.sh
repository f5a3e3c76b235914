for b in 2 64; do for v in "" "CAPSCONV_WK_EY=1" "CAPSCONV_WK_NMW=1" "CAPSCONV_WK_NEPI=2"; do
echo "== B=$b $v"
env $v PROBE=1 timeout 30 python -c "
import sys; sys.argv=['x','layer_s1','$b']; sys.path.insert(0,'tests/probe')
import paper_2104_02621_b200 as pkg
from paper_2104_02621_b200 import _build
pkg.load_library(_build.PROBE_LIB)
import run_cfg; run_cfg.pkg.load_library=lambda *a: None; run_cfg.main()" 2>&1 | grep -E "dI|Error|error" | tail -3
done; done

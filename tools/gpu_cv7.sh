timeout 400 python tools/conv_table.py 2>&1 | tail -26 | cut -c1-100
python - <<'PY'
import sys; sys.path.insert(0,'.')
from paper_2201_12465_b200.gpu import _lib
PY
PB_GEMM_PATH=1 timeout 400 python -c "
import sys; sys.path.insert(0,'.'); sys.argv=['x']
from paper_2201_12465_b200.gpu import _lib
_lib.load().pb_set_gemm_path(1)
sys.path.insert(0,'tools'); import conv_table; conv_table.main()" 2>&1 | tail -26 | cut -c1-100

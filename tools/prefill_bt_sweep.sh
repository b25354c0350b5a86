for bt in 128 160 176 192 224 256; do
  echo "BT $bt"
  ODY_USE_DIAG=1 ODY_PREFILL_BT=$bt timeout 200 python -c "
import os,sys
sys.path.insert(0,'.')
from paper_2311_09550_b200 import _lib as _l
_l.use_diag_library()
import torch
sys.argv=['x']
import tools.prefill_bench as pb
pb.LAYERS=[('o',5120,5120),('down',5120,13824),('qkv',15360,5120)]
pb.main()
" 2>&1 | grep -v "^{" 
done

mkdir -p gpurun_out
cat > /tmp/eig1.py <<'PY'
import sys, torch; sys.path.insert(0,'.')
from paper_1404_2891_b200 import feast as fb
torch.manual_seed(0)
M = torch.randn(128, 128, dtype=torch.complex128, device='cuda'); fb.small_eig(M); torch.cuda.synchronize()
PY
ncu --set full --import-source on --clock-control none -k regex:reduced_eig -o gpurun_out/eig128b python /tmp/eig1.py > gpurun_out/eig_ncu.log 2>&1

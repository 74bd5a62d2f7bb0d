mkdir -p gpurun_out
python -m pytest tests/test_gpu_small_eig.py tests/test_gpu_iterate.py -x -q > gpurun_out/eig_tests.log 2>&1
FEAST_RE_DEBUG=1 python -c "
import sys, torch, time; sys.path.insert(0,'.')
from paper_1404_2891_b200 import feast as fb
for m in (64,128,152):
    M = torch.randn(m, m, dtype=torch.complex128, device='cuda'); fb.small_eig(M); torch.cuda.synchronize()
    t0=time.perf_counter(); fb.small_eig(M); torch.cuda.synchronize(); print(m, (time.perf_counter()-t0)*1e3, 'ms')
" > gpurun_out/eig_dbg.log 2>&1

import sys, ctypes, torch
sys.path.insert(0, '/root/repo')
from paper_2211_12709_b200 import _lib
from paper_2211_12709_b200.partition import block_starts
lib = _lib.load()
grid = tuple(int(v) for v in sys.argv[1].split(','))
ret = tuple(min(16, n) for n in grid)
g = _lib.make_geom(batch=1, c_in=2, c=2, c_out=2, grid=grid, modes=(8,8,8,8), retained=ret, nranks=1, rank=0,
                   dtype=_lib.F32, act=_lib.ACT_GELU, x_starts=block_starts(grid[0],1), ky_starts=block_starts(ret[1],1))
a = torch.randn((1,2)+grid, device='cuda')
out = torch.empty((1,2,grid[0])+ret[1:], dtype=torch.complex64, device='cuda')
rc = lib.dfno_dft_yzt_fwd(ctypes.byref(g), _lib.ptr(a), None, _lib.SRC_RAW, 1.0, _lib.ptr(out), None)
print('rc', rc); torch.cuda.synchronize(); print('ok')

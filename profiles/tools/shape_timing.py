import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2508_02613_b200 import _native as N
from paper_2508_02613_b200 import microstructures as ms
from paper_2508_02613_b200.solver import pcg_device
dev = torch.device("cuda", 0)
lam, mu = ms.lame_from_poisson()
import ast
for shape in ast.literal_eval(os.environ.get("SHAPES", "[(1024, 256, 512)]")):
    g = torch.Generator(device=dev).manual_seed(0)
    rho = (0.01 + torch.rand(shape, dtype=torch.float64, device=dev, generator=g))
    gh = N.GridHandle(3, shape, tuple(s / 512 for s in shape), device=0)
    gh.set_stream(torch.cuda.current_stream().cuda_stream)
    op = N.OpHandle(gh, rho.data_ptr(), lam, mu, where=N.DEVICE)
    green = N.GreenHandle(gh, lam, mu)
    jac = N.JacobiHandle(op)
    rhs = torch.empty((3,) + shape, dtype=torch.float64, device=dev)
    eb = np.array([1.0, 0, 0, 0, 0, 0])
    N.check(N.load().jfftb_assemble_rhs(op.ptr, N.dptr(eb), rhs.data_ptr(), N.DEVICE))
    x = torch.empty_like(rhs)
    for _ in range(2):
        pcg_device(op, "green-jacobi", green, jac, rhs.data_ptr(), x.data_ptr(), -1.0, 10)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pcg_device(op, "green-jacobi", green, jac, rhs.data_ptr(), x.data_ptr(), -1.0, 20)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 20 * 1e3
    gh.profile_start()
    pcg_device(op, "green-jacobi", green, jac, rhs.data_ptr(), x.data_ptr(), -1.0, 10)
    torch.cuda.synchronize()
    st, it = gh.profile_read(stop=True)
    print(shape, "ms/it %.3f" % dt, {k: round(v, 3) for k, v in st.items()} if isinstance(st, dict) else st, flush=True)
    del op, green, jac, gh, rhs, x, rho
    torch.cuda.empty_cache()

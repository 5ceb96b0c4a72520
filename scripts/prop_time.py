import time, sys
sys.path.insert(0, '.')
import paper_1808_06357_b200 as L
from paper_1808_06357_b200 import configs
cfg = configs.CONFIGS["C1"]; lat = configs.lattice(cfg); a, b, c, p = configs.problem(cfg)
S = L.Solver(lat, cfg.eps, a, b, c, p, cfg.sigma); S.set_dt(cfg.dt); S.discretize_initial()
S.step(cfg.m); S.propagate(64, 64); S.propagate(128, 64)
def t(f):
    t0 = time.perf_counter(); f(); return (time.perf_counter() - t0) * 1e3
for rep in range(2):
    print("step(1024)        %.2f ms" % t(lambda: S.step(1024)))
    print("16 x step(64)     %.2f ms" % t(lambda: [S.step(64) for _ in range(16)]))
    print("propagate(1024,64) %.2f ms" % t(lambda: S.propagate(1024, 64)))
    print("propagate(1024,1024) %.2f ms" % t(lambda: S.propagate(1024, 1024)))
    print("propagate(1024,16) %.2f ms" % t(lambda: S.propagate(1024, 16)))

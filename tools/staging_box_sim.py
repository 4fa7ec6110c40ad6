import sys, numpy as np
sys.path.insert(0,'/root/repo')
import bench, oracle
from paper_2501_01628_b200.volume import decompose
def sim(cfg, R, rank, tw, th, stride=7):
    wl = bench.build_workload(cfg, R, "even")
    cam = wl.cams[0]; W,H = wl.W, wl.H
    ca = oracle.camera_array(cam.position, cam.view_dir, cam.up, cam.fov_y, cam.aspect)
    dirs = oracle.primary_dirs(ca, W, H).reshape(H, W, 3)
    lo, hi = [np.array(v, float) for v in wl.dec.boxes[rank]]
    o = np.array(cam.position)
    ext = []
    rng = np.random.default_rng(0)
    for _ in range(400):
        x0 = rng.integers(0, W - tw); y0 = rng.integers(0, H - th)
        d = dirs[y0:y0+th, x0:x0+tw].reshape(-1, 3)
        # slab interval
        with np.errstate(divide='ignore', invalid='ignore'):
            inv = 1.0 / d
            ta = (lo - o) * inv; tb = (hi - o) * inv
        t0 = np.max(np.minimum(ta, tb), axis=1); t1 = np.min(np.maximum(ta, tb), axis=1)
        hit = t1 > np.maximum(t0, 0)
        if hit.sum() < 8: continue
        d = d[hit]; t0 = np.maximum(t0[hit], 0); t1 = t1[hit]
        a = np.argmax(np.abs(d[0])); b, c = [k for k in range(3) if k != a]
        # sample points along rays every 1 voxel, group by slab along a (local coords)
        for i in range(0, 1):
            pass
        ts = np.arange(0, 3600, 1.0)
        P = o[None, None, :] + ts[None, :, None] * d[:, None, :]
        valid = (ts[None, :] >= t0[:, None]) & (ts[None, :] < t1[:, None])
        cell = np.floor(P - lo).astype(int)
        slab = cell[..., a] >> 3
        for K in np.unique(slab[valid])[::5]:
            m = valid & (slab == K)
            if m.sum() < 32: continue
            eb = cell[..., b][m].max() - cell[..., b][m].min() + 2
            ec = cell[..., c][m].max() - cell[..., c][m].min() + 2
            ext.append((eb, ec, m.sum()))
    e = np.array(ext)
    mx = np.maximum(e[:, 0], e[:, 1]); mn = np.minimum(e[:, 0], e[:, 1])
    print(cfg, rank, f"tile {tw}x{th}", "n", len(e), "max-ext pct 50/90/99", np.percentile(mx, [50, 90, 99]), "min-ext p50", np.percentile(mn, 50),
          "box vox/sample p50", np.median(e[:,0]*e[:,1]*10/e[:,2]))
for tw, th in [(4, 8), (8, 8), (16, 16), (8, 16), (32, 8)]:
    sim("c3", 8, 5, tw, th)
for tw, th in [(4, 8), (16, 16)]:
    sim("c2", 1, 0, tw, th)

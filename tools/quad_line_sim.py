"""Host replay of the c2 / c3 rays: 128-byte lines touched per warp-wide quad load of a beam batch under
different quad memory orders (line shapes (lx, ly, lz) of 8 quads).  python tools/quad_line_sim.py 4 8 c2"""
import sys, numpy as np
sys.path.insert(0,'/root/repo')
import bench, oracle
cfg = sys.argv[3] if len(sys.argv) > 3 else 'c2'
wl = bench.build_workload(cfg, 1 if cfg=='c2' else 8, 'even')
cam = wl.cams[0]; W, H = wl.W, wl.H
ca = oracle.camera_array(cam.position, cam.view_dir, cam.up, cam.fov_y, cam.aspect)
dirs = oracle.primary_dirs(ca, W, H).reshape(H, W, 3)
rank = int(sys.argv[4]) if len(sys.argv) > 4 else 0
lo_, hi_ = [np.array(v, float) for v in wl.dec.boxes[rank]]
lo, hi = lo_, hi_
o = np.array(cam.position)
rng = np.random.default_rng(0)
shapes = [(8,1,1),(1,8,1),(1,1,8),(2,4,1),(4,2,1),(2,2,2),(1,4,2),(1,2,4),(2,1,4),(4,1,2),(2,1,4)]
stats = {}
BW, BH = int(sys.argv[1]), int(sys.argv[2])
ntile = 0
for it in range(5000):
    x0 = rng.integers(0, W//BW) * BW; y0 = rng.integers(0, H//BH) * BH
    d = dirs[y0:y0+BH, x0:x0+BW].reshape(-1, 3)
    with np.errstate(divide='ignore', invalid='ignore'):
        inv = 1.0/d; ta = (lo-o)*inv; tb = (hi-o)*inv
    t0 = np.max(np.minimum(ta,tb),1); t1 = np.min(np.maximum(ta,tb),1)
    t0 = np.maximum(t0, 0); hit = t1 > t0
    if hit.sum() < 16: continue
    ntile += 1
    a = int(np.argmax(np.abs(d[np.argmax(hit)])))
    k0 = np.ceil(t0); n = np.where(hit, np.ceil(t1) - k0, 0).astype(int)
    maxn = n.max(); js = np.arange(maxn)
    P = o[None,None,:] + (k0[:,None,None] + js[None,:,None]) * d[:,None,:] - lo[None,None,:]
    cell = np.floor(P).astype(np.int64) + 1
    valid = js[None,:] < n[:,None]
    slab = (cell[..., a] - 1) >> 3
    sl = np.unique(slab[valid])
    for K in sl[::3]:
        m = valid & (slab == K)
        cnt = m.sum(1); first = np.argmax(m, 1); nb = (cnt + 3)//4
        for bi in range(nb.max()):
            for u in range(4):
                lanes = np.where(nb > bi)[0]
                jj = first[lanes] + np.minimum(bi*4+u, cnt[lanes]-1)
                c = cell[lanes, jj]
                for sh in shapes:
                    key = tuple(c // np.array(sh)).__class__
                    q = c // np.array(sh)
                    nl = len(np.unique(q[:,0] + (q[:,1] << 20) + (q[:,2] << 40)))
                    s = stats.setdefault((a, sh), [0, 0]); s[0] += nl; s[1] += 1
    if ntile >= 250: break
tot = {}
for a in range(3):
    row = []
    for sh in shapes:
        s = stats.get((a, sh))
        if s: row.append(f"{sh}:{s[0]/s[1]:.1f}")
        if s:
            t = tot.setdefault(sh, [0,0]); t[0]+=s[0]; t[1]+=s[1]
    print('axis', a, 'n', stats.get((a,shapes[0]),[0,0])[1], ' '.join(row))
print('all', ' '.join(f"{sh}:{t[0]/t[1]:.2f}" for sh, t in tot.items()))

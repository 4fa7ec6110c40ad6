"""Context-only CPU baseline from the REFERENCE itself: the reference's image-assembly step
-- every rank's f64 RGB row tile through `gather_to_root` + `_assemble_tiles` (engine.py:443-456,485,
transport.py:465-475) on its in-process transport -- at 1920x1080 and 3840x2160 with R = 2, 4, 8.  Runs
HERE (imports /root/reference; it does not exist on the GPU box); the numbers are committed in
profiles/r01_ref_gather.md.  Test infrastructure: nothing in the product imports the reference."""
import json
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
import numpy as np

from dprt import engine, transport  # noqa: E402

out = []
for W, H in ((1920, 1080), (3840, 2160)):
    for R in (2, 4, 8):
        def body(ep):
            row0, row1 = engine.assign_pixels(W, H, ep.R)[ep.rank]
            fb = np.full((row1 - row0, W, 3), 0.5)
            times = []
            for _ in range(3):
                transport_barrier = getattr(transport, "barrier", None)
                if transport_barrier:
                    transport_barrier(ep)
                t0 = time.perf_counter()
                tiles = transport.gather_to_root(ep, engine._tile_bytes(row0, row1, fb))
                if ep.rank == 0:
                    engine._assemble_tiles(tiles, W, H)
                times.append(time.perf_counter() - t0)
            return min(times)

        res = transport.run_collective(R, body)
        rec = {"W": W, "H": H, "R": R, "root_ms": res[0] * 1e3}
        out.append(rec)
        print(json.dumps(rec), flush=True)
json.dump(out, open("/tmp/ref_gather.json", "w"))

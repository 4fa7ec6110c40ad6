"""CPU ORACLE for the DVR + sort-last compositing path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs may import this package, and only as the checker (or the timed CPU baseline).  The product package
``paper_2501_01628_b200`` never imports it.

Parity status: camera rays, slab intervals, row ownership, tone map and PPM are pinned to
golden vectors generated from the reference itself (tests/golden/make_golden.py).  DVR arithmetic
(lattice, trilinear, transfer function, front-to-back, ERT, over-compositing) has no counterpart in the
reference -- "parity unpinned" by any reference test -- and is pinned instead by closed-form KATs and
by the bit-exact agreement of two independent restatements here (C ``dvr_oracle.c`` and the scalar
Python loops in ``scalar.py``).
"""

from .dvr import (  # noqa: F401
    OracleBrick,
    build_oracle,
    camera_array,
    composite,
    cycle_frame,
    det_cos,
    generate_field,
    generate_ml,
    kd_leaves,
    kd_order,
    lattice,
    load_oracle,
    max_threads,
    primary_dirs,
    render_brick,
    render_brick_accum,
    render_lattice,
    sample_counts,
    slab,
    tone_map_rgb8,
)

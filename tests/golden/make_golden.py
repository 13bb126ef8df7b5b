#!/usr/bin/env python3
"""Generate the committed golden vectors from the UNMODIFIED reference (oracle/_ref).

Run in the build container (where /root/reference is mounted and `make -C oracle ref` works):

    python tests/golden/make_golden.py

Every case stores its inputs and the reference's outputs of predict(splitck) +
extrapolate_faces (proj/include/ader/predictor.hpp:118-125), computed by the reference library
compiled from /root/reference/proj/src (oracle/Makefile).  Inputs come from the documented
SplitMix64 generator (oracle/stp_oracle.c orc_generate), so they are reproducible.
"""
import json
import zlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402

ELEMS = {2: 4, 3: 4, 4: 4, 5: 3, 6: 3, 7: 2, 8: 2, 9: 1, 10: 1}


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrays)


def main():
    O.build(with_reference=True)
    ref = O.Reference()
    orc = O.Oracle()
    index = {"generator": "oracle/stp_oracle.c orc_generate (dist 0: U[-1,1]) + orc_material_lmr",
             "reference": os.path.basename(ref.path), "cases": []}

    # elastic, per-element material, orders 2..10 (reference cfg.order = nDof)
    for n, E in ELEMS.items():
        q, rcc = orc.generate(0, 1000 + n, n, 0, E)
        lmr = orc.material_lmr(rcc)
        dt = O.cfl_dt(n, rcc[:, 1].max())
        out = ref.stp(n, 9, q, dt, par=lmr, variant="splitck", threads=1)
        gen = ref.stp(n, 9, q, dt, par=lmr, variant="generic", threads=1)
        name = f"elastic_n{n}"
        save(name, q=q, par_rcc=rcc, par_lmr=lmr, dt=np.array(dt), t_start=np.array(0.0),
             qavg=out.qavg, favg=out.favg, face_q=out.face_q, face_f=out.face_f)
        index["cases"].append({"name": name, "n": n, "m": 9, "elements": E, "pde": "elastic per element",
                               "splitck_vs_generic": max(O.per_element_rel_diff(out.qavg, gen.qavg),
                                                         O.per_element_rel_diff(out.face_f, gen.face_f))})

    # the other reference PDEs (proj/include/ader/pde.hpp:62-84), one shared PDE per case
    src = [0.25, 0.5, 0.8, 1, 1.7, 0.3, 0.25]  # PointSourceSpec of test_predictor.cpp:199-206
    other = [
        ("advection_n4_m3", 4, 3, O.PDE_ADVECTION, [1.0, 0.5, 0.25], 0.0),
        ("ncp_advection_n5_m2", 5, 2, O.PDE_NCP_ADVECTION, [1.0, 0.5, 0.25], 0.0),
        ("demo_n3_m6", 3, 6, O.PDE_DEMO, [], 0.0),
        ("demo_n6_m6", 6, 6, O.PDE_DEMO, [], 0.0),
        ("source_only_n3_m4", 3, 4, O.PDE_SOURCE_ONLY, src, 0.2),
        ("source_only_n5_m4", 5, 4, O.PDE_SOURCE_ONLY, src, 0.2),
    ]
    for name, n, m, kind, args, t0 in other:
        rng = np.random.default_rng(zlib.crc32(name.encode()))
        q = rng.uniform(-1, 1, size=(2, n ** 3 * m))
        a = np.zeros(8)
        a[:len(args)] = args
        dt = 0.04 if kind == O.PDE_SOURCE_ONLY else 0.4 / (3.0 * 3.0 * (2 * n - 1))
        out = ref.stp(n, m, q, dt, pde_kind=kind, args=a, t_start=t0, variant="splitck", threads=1)
        save(name, q=q, args=a, dt=np.array(dt), t_start=np.array(t0), qavg=out.qavg, favg=out.favg,
             face_q=out.face_q, face_f=out.face_f)
        index["cases"].append({"name": name, "n": n, "m": m, "elements": 2, "pde_kind": kind})

    # elastic with a point source on a velocity component, per-element material
    n = 4
    q, rcc = orc.generate(0, 77, n, 0, 2)
    lmr = orc.material_lmr(rcc)
    a = np.array([0.3, 0.6, 0.45, 7, 2.0, 0.05, 0.2, 0.0])
    dt = O.cfl_dt(n, rcc[:, 1].max())
    out = ref.stp(n, 9, q, dt, par=lmr, pde_kind=O.PDE_ELASTIC_SOURCE, args=a, t_start=0.1, threads=1)
    save("elastic_source_n4", q=q, par_rcc=rcc, par_lmr=lmr, args=a, dt=np.array(dt), t_start=np.array(0.1),
         qavg=out.qavg, favg=out.favg, face_q=out.face_q, face_f=out.face_f)
    index["cases"].append({"name": "elastic_source_n4", "n": 4, "m": 9, "elements": 2, "pde_kind": 4})

    # basis operators and SplitMix64 sequence of the reference
    basis = {}
    for n in range(1, 11):
        b = ref.basis(n)
        for k, v in b.items():
            basis[f"{k}_{n}"] = v
    save("basis", **basis)
    save("splitmix", seed0=np.array(ref.splitmix(0, 16), dtype=np.uint64),
         seed12345=np.array(ref.splitmix(12345, 64), dtype=np.uint64))
    with open(os.path.join(HERE, "index.json"), "w") as f:
        json.dump(index, f, indent=1)
    print("wrote", len(index["cases"]), "cases")


if __name__ == "__main__":
    main()

"""Generate golden fixtures by importing the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

Writes tests/golden/golden.npz (small KATs and products) and
tests/golden/digests.json (sha256 of config-sized products, SURVEY.md §8(c)
convention: sha256 of the little-endian words of the owned result).
The GPU box never runs this; tests read the committed outputs.
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = os.environ.get("GF2_REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
import gf2mat as g  # noqa: E402
from gf2mat import _reference as ref  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def dig(m):
    return hashlib.sha256(np.ascontiguousarray(m.words, dtype="<u8")
                          .tobytes()).hexdigest()


def main(big: bool):
    out = {}
    # --- generator KATs (core.py:191-208)
    out["kat_random_1x128_s0"] = g.random(1, 128, 0).words.copy()
    out["kat_random_2x65_s7"] = g.random(2, 65, 7).words.copy()
    out["kat_random_37x200_s123"] = g.random(37, 200, 123).words.copy()
    # --- gray codes (graycode.py:38-48), Fig. 1
    for k in range(1, 6):
        gc = g.build_gray(k)
        out[f"gray_code_k{k}"] = np.array(gc.code, dtype=np.int64)
        out[f"gray_changed_k{k}"] = np.array(gc.changed_bit, dtype=np.int64)
    # --- make_table (graycode.py:108-156) on a window source
    pb = g.random(40, 256, 5)
    w = g.window(pb, 3, 64, 9, 130)
    for k in (3, 8):
        tbl = g.CombinationTable(k, w.ncols)
        g.make_table(w, 1, k, tbl)
        out[f"table_k{k}"] = tbl.rows.copy()
    # --- read_bits KATs (core.py:229-248)
    rb = g.random(3, 256, 7)
    kat = []
    for r in range(3):
        for sc, k in [(0, 8), (60, 8), (62, 4), (120, 16), (190, 3), (248, 8)]:
            kat.append((r, sc, k, g.read_bits(rb, r, sc, k)))
    out["read_bits_kat"] = np.array(kat, dtype=np.int64)
    # --- peel_split KATs (strassen.py:66-84)
    rng = np.random.default_rng(11)
    ps = []
    for _ in range(60):
        m, l, n = (int(x) for x in rng.integers(1, 70000, 3))
        cut = int(rng.choice([64, 128, 1024, 2048, 4096]))
        ps.append((m, l, n, cut) + tuple(g.peel_split(m, l, n, cut)))
    for t in [(16384, 16384, 16384, 2048), (4096, 4096, 4096, 1024),
              (10000, 7001, 12345, 2048), (65536, 65536, 65536, 2048),
              (16385, 16385, 16385, 4096), (100, 100, 100, 4096)]:
        ps.append(t + tuple(g.peel_split(*t)))
    out["peel_split_kat"] = np.array(ps, dtype=np.int64)
    # --- products: owned operands, various shapes, via the reference paths
    cases = []
    shapes = [(1, 1, 1), (2, 2, 2), (3, 70, 5), (64, 64, 64), (65, 63, 129),
              (100, 100, 100), (129, 100, 193), (200, 300, 64), (257, 129, 300),
              (300, 1, 300), (1, 300, 1), (511, 513, 257), (1023, 1024, 1025)]
    for i, (m, l, n) in enumerate(shapes):
        sa, sb = 1000 + i, 2000 + i
        a, b = g.random(m, l, sa), g.random(l, n, sb)
        c = g.mul_strassen(a, b, g.MulParams(cutoff=64))
        assert g.equal(c, g.mul_m4rm(a, b, 8))
        out[f"prod_{i}"] = c.words.copy()
        cases.append((i, m, l, n, sa, sb))
    out["prod_cases"] = np.array(cases, dtype=np.int64)
    # --- window operands at odd word offsets (core.py:110-144)
    pa, pb2, pc = g.random(90, 640, 77), g.random(700, 512, 78), g.random(80, 512, 79)
    aw = g.window(pa, 5, 64, 70, 385)       # word offset 1, ragged width
    bw = g.window(pb2, 11, 192, 385, 250)   # word offset 3, ragged width
    out["win_product"] = g.mul_m4rm(aw, bw, 8).words.copy()
    cw = g.window(pc, 3, 64, 70, 250)
    snap = g.copy_out(pc)
    g.add_into(cw, cw, g.mul_strassen(aw, bw, g.MulParams(cutoff=64)))
    out["win_accum_parent"] = pc.words.copy()
    out["win_accum_parent_before"] = snap.words.copy()
    # --- accumulate variant mul_m4rm_into (m4rm.py:150-155)
    a, b, c0 = g.random(150, 333, 91), g.random(333, 200, 92), g.random(150, 200, 93)
    c = g.copy_out(c0)
    g.mul_m4rm_into(c, a, b, 8, 64, 4)
    out["into_result"] = c.words.copy()
    # --- GF2M file bytes and load() error messages (core.py:443-484)
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        fp = os.path.join(td, "m.gf2m")
        g.save(g.random(37, 200, 5), fp)
        good = open(fp, "rb").read()
        out["gf2m_37x200_s5"] = np.frombuffer(good, dtype=np.uint8).copy()
        g.save(g.window(g.random(9, 300, 6), 2, 64, 5, 130), fp)
        out["gf2m_window"] = np.frombuffer(open(fp, "rb").read(), dtype=np.uint8).copy()
        bad = {"truncated": good[:10], "magic": b"GF3M" + good[4:],
               "version": good[:4] + b"\x02" + good[5:], "length": good[:-8]}
        dirty = bytearray(good)
        width = 4
        off = 21 + (3 * width + width - 1) * 8  # row 3, last word, lowest byte
        dirty[off] |= 1
        bad["dirty"] = bytes(dirty)
        msgs = []
        for name, data in bad.items():
            open(fp, "wb").write(data)
            try:
                g.load(fp)
                msgs.append((name, ""))
            except g.FormatError as exc:
                msgs.append((name, str(exc)))
        out["gf2m_error_names"] = np.array([n for n, _ in msgs])
        out["gf2m_error_msgs"] = np.array([m for _, m in msgs])
    # --- structural ops (core.py:344-376) and mul_cubic (cubic.py:76-102)
    a, b = g.random(70, 130, 61), g.random(70, 77, 62)
    out["augment_ragged"] = g.augment(a, b).words.copy()
    out["augment_aligned"] = g.augment(g.random(70, 128, 63), b).words.copy()
    out["stack"] = g.stack(g.random(30, 130, 64), g.random(41, 130, 65)).words.copy()
    out["transpose_70x130"] = g.transpose(a).words.copy()
    out["cubic_200x300x57"] = g.mul_cubic(g.random(200, 300, 66), g.random(300, 57, 67)).words.copy()
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)

    # --- config digests (SURVEY.md §8(c) seed convention 10i+1/2/3)
    digests = {}
    a, b = g.random(1024, 1024, 11), g.random(1024, 1024, 12)
    digests["cfg1"] = dig(g.mul_m4rm(a, b, 8))
    if big:
        t0 = time.time()
        a, b = g.random(4096, 4096, 21), g.random(4096, 4096, 22)
        digests["cfg2"] = dig(g.mul_strassen(a, b, g.MulParams(cutoff=1024, k=8)))
        print("cfg2", time.time() - t0, flush=True)
        t0 = time.time()
        a, b = g.random(16384, 16384, 31), g.random(16384, 16384, 32)
        digests["cfg3"] = dig(g.mul_strassen(a, b))
        print("cfg3", time.time() - t0, flush=True)
    path = os.path.join(HERE, "digests.json")
    prev = json.load(open(path)) if os.path.exists(path) else {}
    prev.update(digests)
    # values computed in the survey from the reference (cfg4 needs the
    # §8(d) Bernoulli generator; cfg5 took 21 min on one core)
    prev.setdefault("cfg4_product", "72d6193db5e210ecbc95b336101f02e506865c85e8421db0a102f1351d104ac6")
    prev.setdefault("cfg4_addmul", "7e550abcedb3535f07c3498f2289b8c7fd521ad72d5d6db640ea922a868812aa")
    prev.setdefault("cfg5_product", "c6e32dc76743798f0eea38f3adde3af4232e1459a576df9b8cb364a2530d22d1")
    prev.setdefault("cfg5_addmul", "ca72f9e2f6cde38ec33dd9271cd6a2ca4758163ca25a39f2da038dfd244a0f16")
    json.dump(prev, open(path, "w"), indent=1, sort_keys=True)
    print(json.dumps(prev, indent=1))


def main_api():
    """golden_api.npz: the drop-in surface beyond the multiply entries --
    schedule_winograd with a mul_cubic stub multiplier (test_strassen.py:
    66-111; the call order, the final C and the scratch buffers X, Y after
    the 22 steps pin the schedule itself), peel_fixup (test_strassen.py:
    114-160), make_table from window sources with a live right edge and a
    narrower refill (test_graycode.py:100-137), default_params / choose_k
    (tuning.py:29-65) and Gray codes up to k = 16 (graycode.py:38-48)."""
    out = {}
    # --- schedule_winograd
    sched = [(128, 128, 128, 2, 3, 64, 64, 64), (70, 256, 128, 4, 5, 35, 128, 64),
             (130, 384, 256, 21, 22, 65, 192, 128)]
    for i, (m, l, n, sa, sb, m2, l2, n2) in enumerate(sched):
        a, b = g.random(m, l, sa), g.random(l, n, sb)
        c = g.random(m, n, 100 + i)                 # junk: every quadrant is overwritten
        x, y = g.random(m2, max(l2, n2), 200 + i), g.random(l2, n2, 300 + i)
        calls = []
        names = {id(c): 0, id(x): 1, id(a): 2, id(b): 3, id(y): 4}

        def mult(cc, aa, bb):
            rec = []
            for w in (cc, aa, bb):
                p = w.parent if isinstance(w, g.MatrixWindow) else w
                ro = w.row_offset if isinstance(w, g.MatrixWindow) else 0
                co = w.col_offset if isinstance(w, g.MatrixWindow) else 0
                rec += [names[id(p)], ro, co, w.nrows, w.ncols]
            calls.append(rec)
            g.copy_into(cc, g.mul_cubic(aa, bb))

        g.schedule_winograd(a, b, c, (x, y), mult)
        assert g.equal(c, g.mul_cubic(a, b))
        out[f"sched{i}_c"] = c.words.copy()
        out[f"sched{i}_x"] = x.words.copy()
        out[f"sched{i}_y"] = y.words.copy()
        out[f"sched{i}_calls"] = np.array(calls, dtype=np.int64)
    out["sched_cases"] = np.array(sched, dtype=np.int64)
    # --- peel_fixup: C's top-left block from the cubic product, rest junk
    peel = [(65, 64, 64, 14, 15, 64, 64, 64), (100, 70, 130, 16, 17, 64, 64, 64),
            (300, 300, 300, 18, 19, 256, 256, 256), (64, 64, 64, 12, 13, 64, 64, 64),
            (200, 333, 70, 23, 24, 128, 256, 64)]
    for i, (m, l, n, sa, sb, m2, l2, n2) in enumerate(peel):
        a, b = g.random(m, l, sa), g.random(l, n, sb)
        c = g.random(m, n, 400 + i)
        g.copy_into(g.window(c, 0, 0, m2, n2),
                    g.mul_cubic(g.window(a, 0, 0, m2, l2), g.window(b, 0, 0, l2, n2)))
        out[f"peel{i}_before"] = c.words.copy()
        g.peel_fixup(c, a, b, m2, l2, n2, g.MulParams(cutoff=64))
        assert ref.first_mismatch(c, ref.naive_product(a, b)) is None
        out[f"peel{i}_c"] = c.words.copy()
    out["peel_cases"] = np.array(peel, dtype=np.int64)
    # --- make_table
    parent = g.random(6, 192, 8)
    win = g.window(parent, 0, 64, 6, 70)
    t = g.CombinationTable(4, 70)
    g.make_table(win, 1, 4, t)
    out["table_win_k4"] = t.matrix.words.copy()
    b = g.random(8, 64, 6)
    t = g.CombinationTable(8, 64)
    g.make_table(b, 0, 8, t)
    g.make_table(b, 0, 3, t)
    out["table_refill_matrix"] = t.matrix.words.copy()       # rows 8.. keep the k=8 fill
    pb = g.random(40, 1000, 9)
    w = g.window(pb, 5, 128, 20, 777)
    t = g.CombinationTable(12, 777)
    g.make_table(w, 3, 12, t)
    out["table_win_k12"] = t.matrix.words.copy()
    # --- tuning rules the drop-in restates
    kat = []
    for l1 in (1, 4096, 32768, 49152, 1 << 20):
        for l2 in (1 << 12, 100000, 1 << 20, 3 << 20, 50 << 20):
            try:
                p = g.default_params(l1, l2)
                kat.append((l1, l2, p.cutoff, p.b_s, p.k, p.t))
            except g.ParameterError:
                kat.append((l1, l2, -1, -1, -1, -1))
    out["default_params_kat"] = np.array(kat, dtype=np.int64)
    from gf2mat.tuning import choose_k
    ck = [(bs, l1, t, nc, choose_k(bs, l1, t, nc if nc else None))
          for bs in (2, 3, 64, 500, 1024, 4096, 65536) for l1 in (1024, 32768)
          for t in (1, 8) for nc in (0, 64, 2048)]
    out["choose_k_kat"] = np.array(ck, dtype=np.int64)
    for k in (6, 9, 12, 16):
        gc = g.build_gray(k)
        out[f"gray_code_k{k}"] = np.array(gc.code, dtype=np.int64)
        out[f"gray_changed_k{k}"] = np.array(gc.changed_bit, dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "golden_api.npz"), **out)
    print("golden_api.npz:", len(out), "arrays")
    # the reference's public names (gf2mat/__init__.py:62-113)
    with open(os.path.join(HERE, "reference_api.json"), "w") as fh:
        json.dump({"version": g.__version__, "__all__": sorted(g.__all__)}, fh, indent=1)


if __name__ == "__main__":
    if "--api" in sys.argv:
        main_api()
    else:
        main(big="--big" in sys.argv)

"""Capture side: interleaved verify steps of a serving
batch captured from device layer tensors, D2H into pinned segments, flushed
to TIDESIG1 shards at the threshold; the shard bytes are parsed by an
independent Python reader of the documented layout, the SPEC byte accounting
is checked against the oracle, and the shards loaded into a training ring are
bit-identical to the captured requests."""
import ctypes as C
import struct

import pathlib

import numpy as np
import pytest

import oracle
from paper_2602_05145_b200 import _lib, api

from test_hsbuf_gpu import H, verify_steps

pytestmark = pytest.mark.gpu


def read_shard(path):
    """Reader of the format documented in proj/include/specsim/draft_trainer.hpp."""
    b = open(path, "rb").read()
    magic, ver, layers, hidden, bpe, n_rec, payload = struct.unpack_from("<8sIIIIQQ", b, 0)
    assert magic == b"TIDESIG1" and ver == 1 and bpe == 2 and payload + 40 == len(b)
    off, out = 40, []
    W = layers * hidden
    a16 = lambda x: (x + 15) // 16 * 16  # noqa: E731
    for _ in range(n_rec):
        sid, alpha, n, width, flags = struct.unpack_from("<qdiiq", b, off)
        assert width == W
        if flags & 2:  # batch record: alpha slot = n_req
            n_req = int(alpha)
            sids = np.frombuffer(b, np.int64, n_req, off + 32)
            cnts = np.frombuffer(b, np.int32, n_req, off + 32 + 8 * n_req)
            f0 = off + 32 + a16(12 * n_req)
            feat = np.frombuffer(b, np.uint16, n * W, f0).reshape(n, W)
            ids = np.frombuffer(b, np.int32, n, f0 + n * W * 2)
            r = 0
            for s_, c_ in zip(sids, cnts):
                out.append((int(s_), -1.0, 0, feat[r:r + c_], ids[r:r + c_]))
                r += c_
            off += a16(32 + a16(12 * n_req) + n * W * 2 + 4 * n)
            continue
        feat = np.frombuffer(b, np.uint16, n * W, off + 32).reshape(n, W)
        ids = np.frombuffer(b, np.int32, n, off + 32 + n * W * 2)
        out.append((sid, alpha, flags, feat, ids))
        off += 32 if n == 0 else a16(32 + n * W * 2 + 4 * n)
    assert off == len(b)
    return layers, hidden, out


def capture_batch(tmp_path, threshold, n_req=6, batched=False):
    import torch
    cap_obj = api.SignalCapture(api.SignalGeometry(H), tmp_path, flush_threshold=threshold)
    reqs = [verify_steps(11, sid, 41 + 17 * sid) for sid in range(n_req)]
    st = np.zeros(4, np.int64)
    bpt = 3 * H * 2
    keep = []
    stream = torch.cuda.Stream()
    step = 0
    with torch.cuda.stream(stream):
        while any(step < len(s) for _, s in reqs):
            # one serving iteration: every unfinished request verifies together
            live = [sid for sid, (_, s) in enumerate(reqs) if step < len(s)]
            if batched:
                # the batch's rows stacked per layer: request j owns rows [4j, 4j + 4)
                rows = 4
                mats = [np.concatenate([reqs[sid][1][step][0][l] for sid in live]) for l in range(3)]
                tl = [torch.from_numpy(m.view(np.int16)).cuda(non_blocking=True) for m in mats]
                keep.append(tl)
                acc_rows = np.concatenate([reqs[sid][1][step][2] + rows * j
                                           for j, sid in enumerate(live)])
                ids = np.concatenate([reqs[sid][1][step][1] for sid in live])
                counts = [len(reqs[sid][1][step][1]) for sid in live]
                cap_obj.append_batch(live, counts, acc_rows, [t.data_ptr() for t in tl],
                                     rows * len(live), H, ids, stream=stream.cuda_stream)
                oracle.lib().orc_extract_signals(C.c_void_p(st.ctypes.data), int(sum(counts)),
                                                 bpt, threshold)
            for sid in live:
                cap, steps = reqs[sid]
                if not batched:
                    layers, ids, idx = steps[step]
                    tl = [torch.from_numpy(l.view(np.int16)).cuda(non_blocking=True) for l in layers]
                    keep.append(tl)
                    cap_obj.append(sid, [t.data_ptr() for t in tl], layers[0].shape[0], H, ids,
                                   idx, stream=stream.cuda_stream)
                    oracle.lib().orc_extract_signals(C.c_void_p(st.ctypes.data), len(ids), bpt,
                                                     threshold)
                if step == len(steps) - 1:
                    cap_obj.end_sample(sid, cap["alpha_s"])
            step += 1
    stats = cap_obj.stats()
    files = cap_obj.close()
    return reqs, st, stats, files


@pytest.mark.parametrize("batched", [False, True])
def test_capture_shards_roundtrip(tmp_path, batched):
    threshold = 1 << 14  # small: several SPEC flushes / shards
    reqs, st, s, files = capture_batch(tmp_path, threshold, batched=batched)
    assert [s["records"], s["bytes"], s["flushes"], s["cumulative_bytes"]] == list(st)
    assert s["bytes"] + s["cumulative_bytes"] == s["records"] * 3 * H * 2
    assert s["samples"] == len(reqs) and s["files"] <= len(files) and len(files) >= s["flushes"] >= 2
    # independent parse: per request, rows in capture order
    got = {}
    alpha = {}
    for f in files:
        layers, hidden, recs = read_shard(f)
        assert (layers, hidden) == (3, H)
        for sid, a, flags, feat, ids in recs:
            g = got.setdefault(sid, ([], []))
            g[0].append(feat)
            g[1].append(ids)
            if flags & 1:
                alpha[sid] = a
    for sid, (cap, _) in enumerate(reqs):
        assert np.array_equal(np.concatenate(got[sid][0]), cap["features"]), sid
        assert np.array_equal(np.concatenate(got[sid][1]), cap["ids"]), sid
        assert alpha[sid] == cap["alpha_s"]
    # training side: shards -> HBM ring, samples contiguous again
    buf = api.HiddenStateBuffer(api.SignalGeometry(H), 1 << 14)
    assert buf.load_shards(files) == len(reqs)
    for sid, (cap, _) in enumerate(reqs):
        f, ids = buf.read_sample(sid)
        assert np.array_equal(f, cap["features"]) and np.array_equal(ids, cap["ids"])
        n, a = buf.sample_info(sid)
        assert n == len(cap["ids"]) and a == cap["alpha_s"]
    buf.close()


def test_load_shards_one_file_at_a_time(tmp_path):
    """Requests straddle the flush boundaries (rows in one shard, completion
    record in a later one): loading the shards one call at a time as they
    appear appends each sample once its end_sample record is read, with all
    its rows, exactly as loading them all at once."""
    reqs, _, s, files = capture_batch(tmp_path, 1 << 14, batched=True)
    assert len(files) >= 3
    buf = api.HiddenStateBuffer(api.SignalGeometry(H), 1 << 14)
    loaded = [buf.load_shards([f]) for f in files]
    assert sum(loaded) == len(reqs)
    assert loaded[0] < len(reqs)  # some requests were still open at the first flush
    for sid, (cap, _) in enumerate(reqs):
        f, ids = buf.read_sample(sid)
        assert np.array_equal(f, cap["features"]) and np.array_equal(ids, cap["ids"])
        assert buf.sample_info(sid) == (len(cap["ids"]), cap["alpha_s"])
    buf.close()


def test_load_shards_rejects_corrupt_request_count(tmp_path):
    """A batch record's request count is bounded by the bytes left before any
    size arithmetic (a corrupt count must not overflow into an out-of-bounds
    read)."""
    import struct
    _, _, _, files = capture_batch(tmp_path, 0, n_req=3, batched=True)
    raw = bytearray(pathlib.Path(files[0]).read_bytes())
    off = 40
    sid, alpha, n, width, flags = struct.unpack_from("<qdiiq", raw, off)
    assert flags & 2  # first record of a batched capture is a batch record
    for bad in (1e300, -1.0, float("nan"), 2.5):
        struct.pack_into("<d", raw, off + 8, bad)
        p = tmp_path / f"bad_{bad}.tsig"
        p.write_bytes(bytes(raw))
        buf = api.HiddenStateBuffer(api.SignalGeometry(H), 1 << 12)
        with pytest.raises(_lib.DomainError):
            buf.load_shards([p])
        buf.close()


def test_capture_default_threshold_single_shard(tmp_path):
    reqs, st, s, files = capture_batch(tmp_path, 0, n_req=3)  # 64 MiB: no SPEC flush
    assert s["flushes"] == 0 and s["bytes"] == s["records"] * 3 * H * 2
    assert len(files) == 1  # close() persists the partial segment


def test_capture_validation(tmp_path):
    with pytest.raises(_lib.DomainError):
        api.SignalCapture(api.SignalGeometry(H), tmp_path / "missing" / "dir")
    c = api.SignalCapture(api.SignalGeometry(H), tmp_path)
    with pytest.raises(_lib.DomainError):
        c.end_sample(1, 1.5)
    with pytest.raises(_lib.DomainError):
        c.append(1, [0, 0, 0], 4, H, [1, 2], [0, 9])  # accepted_idx out of range
    assert c.close() == []  # nothing captured: no shard
    buf = api.HiddenStateBuffer(api.SignalGeometry(2 * H), 1024)
    reqs, _, _, files = capture_batch(tmp_path, 0, n_req=1)
    with pytest.raises(_lib.DomainError):  # geometry mismatch
        buf.load_shards(files)
    bad = tmp_path / "bad.tsig"
    bad.write_bytes(b"NOTASHARD" * 8)
    buf2 = api.HiddenStateBuffer(api.SignalGeometry(H), 1024)
    with pytest.raises(_lib.DomainError):
        buf2.load_shards([bad])
    buf.close()
    buf2.close()

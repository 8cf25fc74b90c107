"""GPU dataset loader (pars_load_dataset) against the reference's own
load_dataset (dataset.cpp:73-173, oracle/_ref): the same records — decoded
prompt bytes, ids, output_len, prompt_len, samples — and, for rejected
files, the same error text."""
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HEADER = '{"embedding_dim":0,"format":"pars.dataset","version":1}'


def _records(rng, n):
    words = ["alpha", "beta", "gamma", "x", "été", "naïve", "\U0001F600",
             "tab\there", 'quo"te', "back\\slash", "new\nline", "/slash/"]
    out = []
    for i in range(n):
        k = int(rng.integers(1, 40))
        text = " ".join(words[int(j)] for j in rng.integers(0, len(words), k))
        rec = {"id": "r%05d" % i, "prompt": text}
        m = i % 5
        if m == 0:
            rec["output_len"] = int(rng.integers(1, 5000))
        elif m == 1:
            rec["output_len_samples"] = [int(v) for v in rng.integers(1, 900, int(rng.integers(1, 6)))]
        elif m == 2:
            s = [int(v) for v in rng.integers(1, 900, 4)]
            rec["output_len_samples"] = s
            rec["output_len"] = (sorted(s)[1] + sorted(s)[2]) // 2
        elif m == 3:
            rec["output_len"] = 7
            rec["prompt_len"] = int(rng.integers(1, 99))
            rec["extra"] = {"nested": [1, 2.5, -3e4, True, None, {"k": "v "}], "s": "\\u"}
        else:
            rec["output_len"] = 3
            rec["meta"] = [[], {}, "x"]
        out.append(rec)
    return out


def _write(path, lines, crlf=False, trailing_newline=True):
    eol = "\r\n" if crlf else "\n"
    body = eol.join(lines) + (eol if trailing_newline else "")
    with open(path, "wb") as f:
        f.write(body.encode("utf-8"))


def _compare(ctx, ref, path, limit=-1):
    from oracle.bind import OracleError
    try:
        want = ref.load_dataset(path, limit)
    except OracleError as e:
        with pytest.raises(Exception) as ei:
            ctx.load_dataset(path, limit)
        assert str(e) == str(ei.value).split(": ", 1)[-1] or str(e) in str(ei.value), \
            (str(e), str(ei.value))
        return None
    got = ctx.load_dataset(path, limit)
    text, offs, ol, pl, ids = got.export()
    assert len(got) == len(want)
    assert offs.tolist() == want.offs.tolist()
    assert text.tobytes() == want.text[:want.offs[-1]].tobytes()
    assert ol.tolist() == want.output_len.tolist()
    assert pl.tolist() == want.prompt_len.tolist()
    assert ids == want.ids()
    for i in range(len(want)):
        assert got.samples(i) == ref.samples(want, i)
    got.free()
    return len(want)


def test_loader_matches_reference_records(ctx, ref, tmp_path):
    rng = np.random.default_rng(3)
    recs = _records(rng, 3000)
    lines = [HEADER] + [json.dumps(r, ensure_ascii=bool(i % 2),
                                   separators=(",", ":") if i % 3 else (", ", ": "))
                        for i, r in enumerate(recs)]
    lines.insert(5, "")  # empty lines are skipped
    lines.insert(9, "")
    p = tmp_path / "d.jsonl"
    _write(p, lines)
    assert _compare(ctx, ref, p) == 3000
    for limit in (0, 1, 7, 2999, 5000):
        _compare(ctx, ref, p, limit)
    # CRLF endings and no trailing newline ('\r' is JSON whitespace after a
    # record; an "empty" CRLF line is a lone '\r', which both loaders reject)
    _write(p, lines, crlf=True, trailing_newline=False)
    assert _compare(ctx, ref, p) is None
    _write(p, [x for x in lines if x], crlf=True, trailing_newline=False)
    assert _compare(ctx, ref, p) == 3000


def test_loader_round_trips_reference_save(ctx, ref, tmp_path):
    ds = ref.synthesize(5000, 11)
    p = tmp_path / "s.jsonl"
    ref.save_dataset(ds, p)
    assert _compare(ctx, ref, p) == 5000


BAD_LINES = [
    '{"id":"a","prompt":"x y","output_len":0}',
    '{"id":"a","prompt":"x y","output_len":3,}',
    '{"id":"a","prompt":"x y","output_len":3.0}',
    '{"id":"a","prompt":"x y","output_len":"3"}',
    '{"id":"a","prompt":"x y"}',
    '{"id":"","prompt":"x y","output_len":3}',
    '{"id":5,"prompt":"x y","output_len":3}',
    '{"prompt":"x y","output_len":3}',
    '{"id":"a","prompt":7,"output_len":3}',
    '[1,2,3]',
    '"just a string"',
    '{"id":"a","prompt":"x\\qy","output_len":3}',
    '{"id":"a","prompt":"x\\ud800y","output_len":3}',
    '{"id":"a","prompt":"x' + chr(1) + 'y","output_len":3}',
    '{"id":"a","prompt":"x' + chr(0xff) + 'y","output_len":3}',
    '{"id":"a","prompt":"   ","output_len":3}',
    '{"id":"a","prompt":"x","output_len_samples":[]}',
    '{"id":"a","prompt":"x","output_len_samples":[3,0]}',
    '{"id":"a","prompt":"x","output_len_samples":[3,5],"output_len":9}',
    '{"id":"a","prompt":"x","output_len":3,"prompt_len":-1}',
    '{"id":"a","prompt":"x","output_len":01}',
    '{"id":"a","prompt":"x","output_len":3} trailing',
    '{"id":"a","prompt":"x","output_len":99999999999999999999}',
    '{"id":"a","prompt":"x","output_len":3,"z":tru}',
    '{"id":"a","prompt":"x","output_len":3',
    chr(13),
]


@pytest.mark.parametrize("k", range(len(BAD_LINES)))
def test_loader_rejects_like_the_reference(ctx, ref, tmp_path, k):
    good = '{"id":"g%d","prompt":"ok ok","output_len":4}'
    lines = [HEADER] + [good % i for i in range(5)] + [BAD_LINES[k]] + [good % 9]
    p = tmp_path / "bad.jsonl"
    with open(p, "wb") as f:
        f.write(("\n".join(lines) + "\n").encode("latin-1"))
    assert _compare(ctx, ref, p) is None


def test_loader_duplicate_ids_and_headers(ctx, ref, tmp_path):
    p = tmp_path / "x.jsonl"
    for lines in (
        [HEADER, '{"id":"a","prompt":"x","output_len":3}', '{"id":"b","prompt":"x","output_len":3}',
         '{"id":"a","prompt":"y","output_len":4}'],
        [HEADER, '{"id":"\\u0061","prompt":"x","output_len":3}', '{"id":"a","prompt":"x","output_len":3}'],
        ['{"format":"other","version":1}', '{"id":"a","prompt":"x","output_len":3}'],
        ['{"format":"pars.dataset","version":2}'],
        ['{"format":"pars.dataset","version":1,"embedding_dim":-1}'],
        ['not json'],
        [HEADER],
    ):
        _write(p, lines)
        _compare(ctx, ref, p)
    open(p, "wb").close()
    _compare(ctx, ref, p)


def test_loader_embedding_records_are_unsupported(ctx, ref, tmp_path):
    from paper_2510_03243_b200 import ParsError
    p = tmp_path / "e.jsonl"
    _write(p, ['{"embedding_dim":2,"format":"pars.dataset","version":1}',
               '{"id":"a","prompt":"x","output_len":3,"embedding":[0.5,1]}'])
    assert len(ref.load_dataset(p)) == 1
    with pytest.raises(ParsError, match="does not parse 'embedding' arrays"):
        ctx.load_dataset(p)


def test_loaded_dataset_scores_like_reference(ctx, ref, tmp_path):
    """The device arena feeds pars_dev_score_text directly: scores equal the
    reference's score_batch over load_dataset's records."""
    import ctypes
    import torch
    from oracle.bind import Extractor as OEx
    from paper_2510_03243_b200 import MODE_EXACT, Extractor, lib
    ds = ref.synthesize(2000, 17)
    p = tmp_path / "s.jsonl"
    ref.save_dataset(ds, p)
    g = ctx.load_dataset(p)
    w = np.random.default_rng(1).normal(size=4096)
    d_w = torch.from_numpy(w).cuda()
    out = torch.zeros(len(g), dtype=torch.float64, device="cuda")
    ex = Extractor.make()
    assert lib().pars_dev_score_text(ctx.h, ctypes.byref(ex), g.dev_text, g.dev_offsets, len(g),
                                     d_w.data_ptr(), 0.0, MODE_EXACT, out.data_ptr(), None) == 0
    torch.cuda.synchronize()
    want = np.zeros(len(ds))
    ref.L.ref_score_batch(ctypes.byref(OEx.make()), ds.h, w.ctypes.data, ctypes.c_double(0.0),
                          want.ctypes.data)
    assert (out.cpu().numpy().view(np.uint64) == want.view(np.uint64)).all()


def test_loader_token_counts_and_escapes_at_every_offset(ctx, ref, tmp_path):
    """prompt_len defaults to the whitespace-token count of the DECODED prompt:
    escaped whitespace (\\t \\n \\r \\f \\u0020 \\u000b) splits tokens, escaped
    non-space does not, and raw UTF-8 / escapes land at every offset
    relative to the parser's 8-byte fast path."""
    rng = np.random.default_rng(17)
    pieces = ["a", "bb", "ccc ", " ", "  ", "\\t", "\\n", "\\r", "\\f", "\\u0020", "\\u000b",
              "\\u00e9", "\\ud83d\\ude00", "\\\"", "\\\\", "\\/", "x" * 13, "é", "中",
              "😀", "\\u0041", "\\b"]
    lines = [HEADER]
    for i in range(4000):
        k = int(rng.integers(0, 60))
        body = "".join(pieces[int(j)] for j in rng.integers(0, len(pieces), k))
        body = " " * int(rng.integers(0, 9)) + body + "z"  # shift the alignment; >= 1 token
        lines.append('{"id":"e%05d","prompt":"%s","output_len":%d}' % (i, body, 1 + i % 7))
    p = tmp_path / "esc.jsonl"
    _write(p, lines)
    assert _compare(ctx, ref, p) == 4000

"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container (the reference is importable read-only):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
Writes tests/golden/*.npz / *.json.  The GPU box never needs /root/reference:
tests read only these committed files.
"""

from __future__ import annotations

import io
import json
import sys
from pathlib import Path
from unittest import mock

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

import walkvec  # noqa: E402
from walkvec import (Triple, build_graph, build_vocabulary, init_embeddings, train, TrainConfig,  # noqa: E402
                     random_walks, bfs_walks, generate_pairs, assign_predicates, gen_barabasi)
from walkvec import walks as ref_walks  # noqa: E402


def rows_graph(rows):
    vocab, edges = build_vocabulary([Triple(s, p, o) for s, p, o in rows])
    return vocab, edges, build_graph(edges, len(vocab))


def random_rows(rng, n_vertices, n_edges, n_predicates=3):
    # same as the reference's tests/conftest.py:56-64 random_edge_rows
    out = []
    for _ in range(n_edges):
        u = int(rng.integers(0, n_vertices))
        v = int(rng.integers(0, n_vertices))
        p = int(rng.integers(0, n_predicates))
        out.append((f"v{u}", f"p{p}", f"v{v}"))
    return out


def philox_patch():
    return mock.patch("numpy.random.default_rng", lambda ss: np.random.Generator(np.random.Philox(ss)))


def seedseq():
    ents = [[42, 0, 0], [42, 0, 7], [7, 0, 244140], [42, 1, 0], [42, 1, 2, 0], [123456789012, 0, 3], [0, 0, 0],
            [2**40 + 5, 1, 1], [3, 0, 2**33 + 9]]
    out = {"entropies": json.dumps(ents)}
    for i, e in enumerate(ents):
        ss = np.random.SeedSequence(e)
        out[f"state4_{i}"] = ss.generate_state(4, np.uint64)
        pcg = np.random.PCG64(np.random.SeedSequence(e))
        out[f"pcg_{i}"] = pcg.random_raw(1100)[[0, 1, 2, 3, 999, 1000, 1099]]
        ph = np.random.Philox(np.random.SeedSequence(e))
        out[f"philox_{i}"] = ph.random_raw(1100)[[0, 1, 2, 3, 4, 5, 999, 1000, 1099]]
    np.savez_compressed(OUT / "seedseq.npz", **out)


def walks():
    cases = {}
    specs = [  # (graph seed, n_vertices, n_edges, depth, number, walk seed, root repeat, dup_free)
        (11, 40, 200, 4, 1, 9, 410, False),      # > 2 shards incl. partial (reference worker test shape)
        (12, 25, 100, 5, 3, 21, 1, False),
        (0, 30, 120, 6, 4, 0, 1, False),
        (3, 60, 90, 8, 7, 5, 1, False),          # sparse: many sinks / early termination
        (4, 15, 40, 3, 500, 3, 1, True),         # duplicate_free
        (5, 200, 700, 1, 2, 17, 1, False),
        (6, 500, 1500, 8, 40, 123456789012, 1, False),  # 2-word seed, 20000 walks
    ]
    for ci, (gs, nv, ne, depth, number, seed, rep, dup) in enumerate(specs):
        rng = np.random.default_rng(gs)
        vocab, edges, g = rows_graph(random_rows(rng, nv, ne))
        roots = np.repeat(vocab.entity_tokens(), rep)[: ref_walks.SHARD_SIZE * 2 + 17] if rep > 1 \
            else vocab.entity_tokens()
        c = random_walks(g, roots, walk_depth=depth, walk_number=number, rng_seed=seed, duplicate_free=dup)
        with philox_patch():
            cp = random_walks(g, roots, walk_depth=depth, walk_number=number, rng_seed=seed, duplicate_free=dup)
        cases[f"c{ci}_edges"] = edges
        cases[f"c{ci}_V"] = np.array(len(vocab))
        cases[f"c{ci}_roots"] = roots
        cases[f"c{ci}_params"] = np.array([depth, number, seed % (2**62), int(dup)], dtype=np.int64)
        cases[f"c{ci}_seed"] = np.array(str(seed))
        cases[f"c{ci}_pcg_tokens"] = c.tokens
        cases[f"c{ci}_pcg_offsets"] = c.offsets
        cases[f"c{ci}_philox_tokens"] = cp.tokens
        cases[f"c{ci}_philox_offsets"] = cp.offsets
        cases[f"c{ci}_row_offsets"] = g.row_offsets
        cases[f"c{ci}_col_targets"] = g.col_targets
        cases[f"c{ci}_col_predicates"] = g.col_predicates
    cases["n_cases"] = np.array(len(specs))
    np.savez_compressed(OUT / "walks.npz", **cases)


def bfs():
    cases = {}
    rng = np.random.default_rng(77)
    ci = 0
    for trial in range(24):
        n = int(rng.integers(4, 120))
        ne = int(rng.integers(n, 4 * n))
        if trial % 2 == 0:  # DAG like test_acceptance._random_dag_rows
            order = rng.permutation(n)
            rows = []
            for _ in range(ne):
                a, b = rng.integers(0, n, size=2)
                if a == b:
                    continue
                u, v = (a, b) if order[a] < order[b] else (b, a)
                rows.append((f"v{u}", f"p{int(rng.integers(0, 3))}", f"v{v}"))
        else:
            rows = random_rows(rng, n, ne)
        if not rows:
            continue
        vocab, edges, g = rows_graph(rows)
        depth = int(rng.integers(1, 7))
        roots = vocab.entity_tokens()
        corpus, table = bfs_walks(g, roots, depth)
        cases[f"c{ci}_edges"] = edges
        cases[f"c{ci}_V"] = np.array(len(vocab))
        cases[f"c{ci}_depth"] = np.array(depth)
        cases[f"c{ci}_roots"] = roots
        cases[f"c{ci}_tokens"] = corpus.tokens
        cases[f"c{ci}_offsets"] = corpus.offsets
        cases[f"c{ci}_table"] = np.array(table.rows(), dtype=np.int64).reshape(-1, 3)
        ci += 1
    cases["n_cases"] = np.array(ci)
    np.savez_compressed(OUT / "bfs.npz", **cases)


def embeddings_and_train():
    out = {}
    inp = init_embeddings(37, 13, 5)
    out["init_in"], out["init_out"] = inp.input_matrix, inp.output_matrix
    # pairs with min_count filtering (windows close over gaps)
    rng = np.random.default_rng(3)
    seqs = [rng.integers(0, 12, size=int(rng.integers(1, 9))) for _ in range(60)]
    lens = np.array([len(s) for s in seqs])
    toks = np.concatenate(seqs)
    offs = np.concatenate([[0], np.cumsum(lens)])
    corpus = walkvec.WalkCorpus(toks, offs, "random")
    pairs, freq = generate_pairs(corpus, 3, 6, 12)
    out["pairs_tokens"], out["pairs_offsets"], out["pairs"], out["pairs_freq"] = toks, offs, pairs, freq
    # train cases on a small random-walk corpus
    vocab, edges, g = rows_graph(random_rows(np.random.default_rng(21), 30, 150, 4))
    c = random_walks(g, vocab.entity_tokens(), walk_depth=4, walk_number=6, rng_seed=4)
    out["train_tokens"], out["train_offsets"], out["train_V"] = c.tokens, c.offsets, np.array(len(vocab))
    cfgs = {
        "sparse": dict(min_count=2, vector_size=12, epochs=2, window_size=3, negative_samples=4, learning_rate=0.02,
                       batch_size=64),
        "dense": dict(min_count=0, vector_size=8, epochs=1, window_size=2, negative_samples=2, learning_rate=0.01,
                      batch_size=128, use_sparse=False),
        "auto": dict(min_count=10, vector_size=16, epochs=1, window_size=5, negative_samples=5),
        "multi": dict(min_count=0, vector_size=8, epochs=2, window_size=2, negative_samples=2, workers=2,
                      reproducible=True, batch_size=16),
        "multi3": dict(min_count=1, vector_size=6, epochs=1, window_size=3, negative_samples=1, workers=3,
                       reproducible=True, batch_size=10),
    }
    for name, kw in cfgs.items():
        model, losses = train(c, len(vocab), TrainConfig(**kw), 42)
        out[f"{name}_in"], out[f"{name}_out"] = model.input_matrix, model.output_matrix
        out[f"{name}_losses"] = np.array(losses)
        out[f"{name}_touched_in"], out[f"{name}_touched_out"] = model.touched_input, model.touched_output
        out[f"{name}_cfg"] = np.array(json.dumps(kw))
    np.savez_compressed(OUT / "w2v.npz", **out)


def cbow():
    """CBOW (w2v.py:194-222 instances, :302-361 gradients): instance tables and train() runs."""
    from walkvec.w2v import generate_cbow_instances

    out = {}
    rng = np.random.default_rng(3)
    seqs = [rng.integers(0, 12, size=int(rng.integers(1, 9))) for _ in range(60)]
    lens = np.array([len(s) for s in seqs])
    toks = np.concatenate(seqs)
    offs = np.concatenate([[0], np.cumsum(lens)])
    corpus = walkvec.WalkCorpus(toks, offs, "random")
    ctx, lengths, targets, freq = generate_cbow_instances(corpus, 3, 6, 12)
    out["inst_tokens"], out["inst_offsets"] = toks, offs
    out["inst_ctx"], out["inst_lengths"], out["inst_targets"], out["inst_freq"] = ctx, lengths, targets, freq
    vocab, edges, g = rows_graph(random_rows(np.random.default_rng(21), 30, 150, 4))
    c = random_walks(g, vocab.entity_tokens(), walk_depth=4, walk_number=6, rng_seed=4)
    out["train_tokens"], out["train_offsets"], out["train_V"] = c.tokens, c.offsets, np.array(len(vocab))
    cfgs = {
        "sparse": dict(model="cbow", min_count=2, vector_size=12, epochs=2, window_size=3, learning_rate=0.02,
                       batch_size=64),
        "dense": dict(model="cbow", min_count=0, vector_size=8, epochs=1, window_size=2, learning_rate=0.01,
                      batch_size=128, use_sparse=False),
        "auto": dict(model="cbow", min_count=10, vector_size=16, epochs=1, window_size=5),
        "multi": dict(model="cbow", min_count=0, vector_size=8, epochs=2, window_size=2, workers=2,
                      reproducible=True, batch_size=16),
    }
    for name, kw in cfgs.items():
        model, losses = train(c, len(vocab), TrainConfig(**kw), 42)
        out[f"{name}_in"], out[f"{name}_out"] = model.input_matrix, model.output_matrix
        out[f"{name}_losses"] = np.array(losses)
        out[f"{name}_touched_in"], out[f"{name}_touched_out"] = model.touched_input, model.touched_output
        out[f"{name}_cfg"] = np.array(json.dumps(kw))
    np.savez_compressed(OUT / "cbow.npz", **out)


def ingest_cases():
    """N-Triples and edge-table inputs through the reference's parse + build_vocabulary
    (ingest.py:116-257, 368-396): tokens, lexicals, roles, edges and errors."""
    import tempfile

    from walkvec.ingest import ParseError, parse_edge_table, parse_ntriples

    good = (
        '<http://x/a> <http://x/p> <http://x/b> .\n'
        '# a comment line\n'
        '\n'
        '_:b1 <http://x/p> "lit \\"q\\" \\u00e9" .\r\n'
        '<http://x/b>\t<http://x/q> "12"^^<http://www.w3.org/2001/XMLSchema#int> . # tail comment\r'
        '<http://x/\\u0063> <http://x/p> "hello"@en-GB .\n'
        '<http://x/p> <http://x/q> <http://x/c> .\n'
        '  <http://x/c> <http://x/p> _:b1 .\n'
        '<http://x/é> <http://x/p> <http://x/a> .\n'
        '<_:b1> <http://x/q> "x\\ty" .'
    )
    bad_lines = [
        '<http://x/a> <http://x/p> <http://x/b>',
        '<http://x/a <http://x/p> <http://x/b> .',
        '_: <http://x/p> <http://x/b> .',
        '<http://x/a> <http://x/p> "open .',
        '<http://x/a> <http://x/p> "v"^^http://t .',
        '<http://x/a> <http://x/p> "v"^^<http://t .',
        '<http://x/a> <http://x/p> "v"@ .',
        '<http://x/a> <http://x/p> ?x .',
        '"s" <http://x/p> <http://x/b> .',
        '<http://x/a> _:p <http://x/b> .',
        '<http://x/a> <http://x/p> <http://x/b> . junk',
        '<http://x/a> <http://x/p> "bad \\q" .',
        '<http://x/a> <http://x/p> "bad \\u12" .',
        '<http://x/a> <http://x/p> "bad \\uZZZZ" .',
        '<http://x/a> <http://x/p> "bad \\U00110000" .',
        '<http://x/a> <http://x/p>',
    ]
    cases = []
    for include in (False, True):
        vocab, edges = build_vocabulary(parse_ntriples(io.BytesIO(good.encode())), include_literals=include)
        cases.append(dict(name=f"good_lit{int(include)}", format="nt", text=good, include_literals=include,
                          strict=False, lexicals=vocab.lexical_of, edges=edges.tolist(),
                          entities=vocab.entity_tokens().tolist(), predicates=sorted(vocab._predicate_tokens)))
    mixed = "\n".join(["<http://x/a> <http://x/p> <http://x/b> ."] + bad_lines + ["<http://x/b> <http://x/p> <http://x/z> ."])
    sink = []
    vocab, edges = build_vocabulary(parse_ntriples(io.BytesIO(mixed.encode()), error_sink=sink))
    cases.append(dict(name="mixed_nonstrict", format="nt", text=mixed, include_literals=False, strict=False,
                      lexicals=vocab.lexical_of, edges=edges.tolist(), entities=vocab.entity_tokens().tolist(),
                      predicates=sorted(vocab._predicate_tokens),
                      errors=[[e.line, e.reason] for e in sink]))
    for i, line in enumerate(bad_lines):
        text = "<http://x/a> <http://x/p> <http://x/b> .\n" + line + "\n"
        try:
            build_vocabulary(parse_ntriples(io.BytesIO(text.encode()), strict=True))
            raise AssertionError("expected a ParseError")
        except ParseError as e:
            cases.append(dict(name=f"strict_{i}", format="nt", text=text, strict=True, include_literals=False,
                              error=[e.line, e.reason]))
    try:
        build_vocabulary(parse_ntriples(io.BytesIO(b"<> <http://x/p> <http://x/b> .\n")))
    except ValueError as e:
        cases.append(dict(name="value_error", format="nt", text="<> <http://x/p> <http://x/b> .\n", strict=False,
                          include_literals=False, value_error=str(e)))
    tables = {
        "csv": "s,p,o\na,r,b\nb,r,c\n\nc,q,a\r\na,q,c",
        "tsv": "a\tr\tb\nb\tq\tc\n",
        "txt": "a r b\n\n  b  q\tc \nc r a\n",
    }
    for fmt, text in tables.items():
        for header in (False, True):
            with tempfile.NamedTemporaryFile("w", suffix="." + fmt, delete=False, newline="") as fh:
                fh.write(text)
            vocab, edges = build_vocabulary(parse_edge_table(fh.name, format=fmt, has_header=header))
            cases.append(dict(name=f"table_{fmt}_{int(header)}", format=fmt, text=text, has_header=header,
                              strict=False, include_literals=False, lexicals=vocab.lexical_of, edges=edges.tolist(),
                              entities=vocab.entity_tokens().tolist(), predicates=sorted(vocab._predicate_tokens)))
    with tempfile.NamedTemporaryFile("w", suffix=".csv", delete=False, newline="") as fh:
        fh.write("a,r,b\nb,r\n")
    try:
        build_vocabulary(parse_edge_table(fh.name, format="csv"))
    except ParseError as e:
        cases.append(dict(name="table_columns", format="csv", text="a,r,b\nb,r\n", strict=False,
                          include_literals=False, error=[e.line, e.reason]))
    rows = [("a b", "p>q", "c\\d", "resource"), ("_:b1", "p>q", 'say "hi"\nnow', "literal"),
            ("c\\d", "r", "a b", "resource"), ("é", "p>q", "_:b1", "resource"), ("x", "r", "é", "literal"),
            ("<y>", "r", "x", "resource")]
    for include in (False, True):
        vocab, edges = build_vocabulary([Triple(s_, p_, o_, k_) for s_, p_, o_, k_ in rows],
                                        include_literals=include)
        cases.append(dict(name=f"triples_lit{int(include)}", triples=rows, include_literals=include,
                          lexicals=vocab.lexical_of, edges=edges.tolist(), entities=vocab.entity_tokens().tolist(),
                          predicates=sorted(vocab._predicate_tokens)))
    # quoted csv / tsv (csv.reader, ingest.py:241): delimiters, doubled quotes, line breaks inside
    # quotes (records spanning lines: row numbers are csv.reader's line_num), text after a closing
    # quote, literal quotes inside unquoted fields, an unterminated quote at EOF, headers
    quoted = {
        "q_csv": ('s,p,o\n"a,1",r,"b ""x"" c"\n"multi\nline",r,b\r\nb,"q\r\nz",c\n\n'
                  'c,"r"tail,a"b\n"",r,"""q"""\n'.replace('"",r,"""q"""', 'd,r,"""q"""')),
        "q_tsv": 'a\t"p\tq"\tb\n"x\ny"\tr\t"a"\nb\t"r"\tc,"d"\n',
        "q_empty_subject": 'a,r,b\n"",r,c\n',
        "q_csv_eof": 'a,r,b\nc,r,"open,to\nend',
        "q_header_multi": '"h1\nh2",p,o\na,r,b\n',
    }
    for name, text in quoted.items():
        fmt = "tsv" if "tsv" in name else "csv"
        for header in (False, True):
            with tempfile.NamedTemporaryFile("w", suffix="." + fmt, delete=False, newline="") as fh:
                fh.write(text)
            try:
                vocab, edges = build_vocabulary(parse_edge_table(fh.name, format=fmt, has_header=header))
                cases.append(dict(name=f"{name}_{int(header)}", format=fmt, text=text, has_header=header,
                                  strict=False, include_literals=False, lexicals=vocab.lexical_of,
                                  edges=edges.tolist(), entities=vocab.entity_tokens().tolist(),
                                  predicates=sorted(vocab._predicate_tokens)))
            except ParseError as e:
                cases.append(dict(name=f"{name}_{int(header)}", format=fmt, text=text, has_header=header,
                                  strict=False, include_literals=False, error=[e.line, e.reason]))
            except ValueError as e:
                cases.append(dict(name=f"{name}_{int(header)}", format=fmt, text=text, has_header=header,
                                  strict=False, include_literals=False, value_error=str(e)))
    bad_rows = 'a,r,b\n"x\ny",r\nc,r,d\n'  # a 2-column record spanning lines 2-3: ParseError at line 3
    with tempfile.NamedTemporaryFile("w", suffix=".csv", delete=False, newline="") as fh:
        fh.write(bad_rows)
    try:
        build_vocabulary(parse_edge_table(fh.name, format="csv"))
    except ParseError as e:
        cases.append(dict(name="q_columns_multiline", format="csv", text=bad_rows, strict=False,
                          include_literals=False, error=[e.line, e.reason]))
    (OUT / "ingest.json").write_text(json.dumps(cases, indent=1, ensure_ascii=False) + "\n")


def formats():
    """Reference writers (pipeline.py:236-251, walks.py:344-364): exact output bytes."""
    import base64
    import tempfile

    from walkvec import walks as rw
    from walkvec.pipeline import save_embeddings_text, save_embeddings_tsv

    rng = np.random.default_rng(11)
    special = [0.0, -0.0, 1.0, 0.1, 1e-5, 1.2345678e-5, 123456.78, 12345678.9, 99999999.5, 9.999999995e-05,
               0.00012345678, -3.25e-10, 1e-30, 0.125, 2.5e-07, -7.77777775, 1e15, 4.4999999949999995]
    mats = {"f64": np.concatenate([np.array(special + [0.0] * (-len(special) % 6)),
                                   rng.normal(0, 0.3, 6 * 40) * 10.0 ** rng.integers(-9, 4, 6 * 40)]).reshape(-1, 6)}
    mats["f32"] = rng.normal(0, 0.2, (30, 5)).astype(np.float32).astype(np.float64)
    out = {}
    for name, m in mats.items():
        lex = [f"tok {i}\twith\\ é" if i % 3 == 0 else f"http://x/{i}" for i in range(len(m))]

        class V:
            def lexical(self, t):
                return lex[t]

        for kind, fn in (("text", save_embeddings_text), ("tsv", save_embeddings_tsv)):
            with tempfile.NamedTemporaryFile(delete=False) as fh:
                path = fh.name
            fn(m, V(), path)
            out[f"{name}_{kind}"] = base64.b64encode(open(path, "rb").read()).decode()
        out[f"{name}_matrix"] = m.tolist()
        out[f"{name}_lexicals"] = lex
    toks = rng.integers(0, 50, 40)
    offs = [0, 5, 5, 12, 20, 33, 40]
    corpus = rw.WalkCorpus(toks, np.array(offs), rw.BFS, rw.ENTITY)
    with tempfile.NamedTemporaryFile(delete=False) as fh:
        path = fh.name
    rw.save_corpus_binary(corpus, path)
    out["wvc1"] = base64.b64encode(open(path, "rb").read()).decode()
    out["wvc1_tokens"], out["wvc1_offsets"] = toks.tolist(), offs
    # Vocabulary.save_tsv (ingest.py:307-323): escaped lexicals, roles, frequencies
    from walkvec.ingest import Vocabulary

    voc = Vocabulary()
    lexs = ["http://a/0", "tab\there", "new\nline", "back\\slash", "cr\rx", "é ü 漢", "", "p:knows", "plain"]
    for i, lx in enumerate(lexs):
        (voc._intern_predicate if i in (1, 7) else voc._intern_entity)(lx)
    voc._intern_predicate("plain")  # entity and predicate
    voc.frequency = np.array([3, 0, 7, 12, 1, 0, 5, 100, 2], dtype=np.int64)
    with tempfile.NamedTemporaryFile(delete=False) as fh:
        path = fh.name
    voc.save_tsv(path)
    out["vocab_tsv"] = base64.b64encode(open(path, "rb").read()).decode()
    out["vocab_lexicals"] = lexs
    out["vocab_entities"] = sorted(voc._entity_tokens)
    out["vocab_predicates"] = sorted(voc._predicate_tokens)
    out["vocab_frequency"] = voc.frequency.tolist()
    (OUT / "formats.json").write_text(json.dumps(out, ensure_ascii=False) + "\n")


def pipeline_cases():
    """Reference load_data + fit_transform end to end (pipeline.py:117-219) on a small .nt graph."""
    import tempfile

    from walkvec.pipeline import PipelineConfig, fit_transform, load_data

    rng = np.random.default_rng(8)
    lines = []
    for _ in range(400):
        u, v, p_ = int(rng.integers(0, 60)), int(rng.integers(0, 60)), int(rng.integers(0, 5))
        lines.append(f"<http://kg/e{u}> <http://kg/p{p_}> <http://kg/e{v}> .")
    lines += ['<http://kg/e1> <http://kg/label> "one"@en .', "_:b <http://kg/p1> <http://kg/e2> ."]
    text = "\n".join(lines) + "\n"
    with tempfile.NamedTemporaryFile("w", suffix=".nt", delete=False) as fh:
        fh.write(text)
    configs = {
        "sg_random": dict(walk_depth=3, walk_number=6, vector_size=8, epochs=2, min_count=1, window_size=2,
                          negative_samples=3, batch_size=128),
        "cbow_bfs_entity": dict(walk_strategy="bfs", walk_depth=2, embedding_model="cbow", vector_size=8, epochs=1,
                                min_count=2, window_size=2, batch_size=64, projection="entity"),
        "sg_random_dupfree_property": dict(walk_depth=4, walk_number=5, duplicate_free=True, vector_size=6,
                                           epochs=1, min_count=1, window_size=3, negative_samples=2,
                                           projection="property", batch_size=100),
    }
    out = {"text": text, "cases": {}}
    for name, kw in configs.items():
        vocab, edges = load_data(fh.name)
        table = fit_transform(edges, vocab, PipelineConfig(**kw))
        out["cases"][name] = dict(cfg=kw, lexicals=vocab.lexical_of, vectors=table.vectors.tolist(),
                                  losses=list(table.losses), trained=table.trained_mask.tolist(),
                                  frequency=vocab.frequency.tolist())
    (OUT / "pipeline.json").write_text(json.dumps(out) + "\n")


def two_clique():
    rows = []
    for base in ("x", "y"):
        members = [f"{base}{i}" for i in range(5)]
        rows += [(u, "p", v) for u in members for v in members if u != v]
    rows.append(("x0", "p", "y0"))
    vocab, edges, g = rows_graph(rows)

    def band(dim):
        res = []
        for seed in range(10):
            corpus = random_walks(g, vocab.entity_tokens(), walk_depth=4, walk_number=25, rng_seed=42 + seed)
            cfg = TrainConfig(min_count=1, vector_size=dim, epochs=10, learning_rate=0.01, window_size=5,
                              negative_samples=5)
            model, losses = train(corpus, len(vocab), cfg, 42 + seed)
            v = model.input_matrix
            x = [vocab.token_of[f"x{i}"] for i in range(5)]
            y = [vocab.token_of[f"y{i}"] for i in range(5)]

            def cos(a, b):
                return float(np.dot(v[a], v[b]) / (np.linalg.norm(v[a]) * np.linalg.norm(v[b])))

            intra = [cos(a, b) for grp in (x, y) for a in grp for b in grp if a < b]
            inter = [cos(a, b) for a in x for b in y]
            res.append(dict(seed=42 + seed, margin=float(np.mean(intra) - np.mean(inter)), loss0=losses[0],
                            loss_last=losses[-1]))
        return res

    # d 16 (the reference's own acceptance setting) and d 200 (the benchmark's width)
    (OUT / "two_clique.json").write_text(json.dumps(dict(edges=edges.tolist(), V=len(vocab),
                                                         x=[vocab.token_of[f"x{i}"] for i in range(5)],
                                                         y=[vocab.token_of[f"y{i}"] for i in range(5)],
                                                         roots=vocab.entity_tokens().tolist(), runs=band(16),
                                                         runs_d200=band(200)), indent=1))


def vocab_encoding():
    e2 = gen_barabasi(300, 3, seed=7)
    triples = assign_predicates(e2, 5, seed=7)
    vocab, edges = build_vocabulary(triples)
    picks = np.array([int(t.predicate[1:]) for t in triples])
    np.savez_compressed(OUT / "vocab.npz", raw=e2, picks=picks, edges=edges, entity_tokens=vocab.entity_tokens(),
                        V=np.array(len(vocab)))


if __name__ == "__main__":
    # python make_golden.py [generator ...]   (default: all)
    gens = {f.__name__: f for f in (seedseq, walks, bfs, embeddings_and_train, two_clique, vocab_encoding, cbow,
                                    ingest_cases, formats, pipeline_cases)}
    for name in (sys.argv[1:] or list(gens)):
        gens[name]()
    for p in sorted(OUT.glob("*.np*")) + sorted(OUT.glob("*.json")):
        print(p.name, p.stat().st_size)

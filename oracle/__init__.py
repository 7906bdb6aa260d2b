"""Float64 CPU oracle for the NPM hot path (arXiv 2504.04315).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2504_04315_b200``) never imports it, and
this package imports nothing from the product path: the two share no code.

Citation convention: ``P:n`` = line n of the paper's LaTeX source
(``PAPER.md``), with the section / equation named alongside; ``S:n`` = line n of
the CPU-program specification (``SPEC.md``), used only where the paper is
silent; ``C-xx`` = the reading recorded in ``SURVEY.md`` §8(c) and DESIGN.md.

Every function here is plain, slow and written in the paper's order and
notation.  Floating point is float64 except where a reading (C-A1) pins an
fp32 sequence that decides an integer (the grid cell index), which both sides
then compute in fp32.

Pins (tests/test_oracle_*.py) tie each function to something other than
itself: closed forms, quadrature, finite differences, chi-square against the
pdf, brute force on tiny grids, published Philox known-answer vectors.
One function is **parity unpinned** against the paper: the spatial hash of
hashed grid levels (C-A4) -- the paper names no hash; it is pinned only to our
declared convention.

Modules
-------
philox  Philox4x32-10 counter-based generator (C-O11)
grid    multi-resolution grid encoding, Eq. 13 (C-O1..C-O5, C-O15)
sh      real spherical harmonics, 4 bands (C-O6)
mlp     decoder MLP, Eq. 14 (C-O7, C-O14)
vmf     Table 1 mappings, Eq. 3/4 pdf, Jakob sampling, Eq. 9 gradient head
        (C-O8..C-O13)
adam    Adam + EMA (C-O17, C-O18)
npm     the model: encode / decode / pdf / sample / train_step
guide   one-sample MIS of BSDF and guide, training-record unwind (f-1)
product closed-form vMF product, cosine-lobe factorisation (f-2)
"""

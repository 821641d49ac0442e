"""CPU oracle for V-/I-TiMePReSt — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct numpy (fp64) implementation of what the hot
path computes, written from PAPER.md (arXiv 2509.23241).  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may import it.  The product path (`paper_2509_23241_b200`) never imports,
links or executes anything here, and this package never imports the product.

Modules (each function cites the passage it follows; P:n = PAPER.md line n,
S:n = SPEC.md line n, Z# = DESIGN.md reading):
  bf16       -- round-to-nearest-even bfloat16 storage emulation (Z13)
  tf32       -- round-to-nearest (ties away) tf32 storage emulation (tf32 mode, Z28)
  staleness  -- f(δ) = e^{-λδ} (Eq. 2), Eq. 1 factor, blend coeffs (Z1)
  schedule   -- static nF1B per-stage event order (Z6, Z7)
                and a dependency-driven executor
  mlp        -- Linear/ReLU/softmax-CE stage math, SGD/momentum update
  pipeline   -- whole-pipeline replay of V- and I-TiMePReSt

Parity status: every function is pinned by a `-m "not gpu"` test in
tests/test_oracle_*.py against values the paper prints, closed forms, brute
force, finite differences or an independent library routine (torch autograd,
torch.optim.SGD, ml_dtypes).  No function is "parity unpinned".
"""

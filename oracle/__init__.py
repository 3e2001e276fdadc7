"""CPU oracle for the packed-jobs hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline.  The product (``paper_2410_22254_b200``) never imports
it; its hot path is the sm_100a library ``libtlk.so`` and fails loudly when
that library is missing.

What it restates
----------------
* Slot mapping (triples core / plan / executor semantics): the reference
  itself is the oracle here -- ``tests/golden/mapping.json`` is generated from
  ``/root/reference/pkg/src/trilaunch`` by ``tests/golden/gen_mapping_golden.py``
  (PINNED: bit-exact against the reference's own outputs).
* The training tasks (reference: absent -- the reference runs them as opaque
  argv, executor.py:199; PAPER.md:96-101 names PyTorch models).
  ``oracle.models`` restates them in numpy fp32: MNIST MLP 784-512-512-10 and
  the pytorch/examples MNIST CNN without dropout, Adam/AdamW/SGD.  The
  reference pins no loss/weight values, so this restatement is PINNED instead
  against PyTorch CPU (the framework the paper's jobs use) via
  ``tests/golden/gen_torch_golden.py`` -> ``tests/golden/torch_*.npz``.

Numerics contract (shared with the CUDA path):
GEMM operands are bf16 (round-to-nearest-even) with fp32 accumulation; the
oracle's ``bf16=True`` mode rounds exactly the tensors the GPU rounds, so GPU
and oracle differ only by fp32 summation order.  ``bf16=False`` is plain fp32
and is what the PyTorch pinning uses.
"""

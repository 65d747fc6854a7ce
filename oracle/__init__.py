"""CPU oracle for the ParaGAN replicated BigGAN training step.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import or run
anything in this package.  The product path (``paper_2411_03999_b200`` + ``libparagan.so``)
never imports it, and the oracle never imports the product: the two share no
code, tables or constants.  Only the seeded input generators
(``paper_2411_03999_b200/inputs.py``, which hold none of the method's arithmetic) feed
both sides.

Everything here is plain PyTorch CPU arithmetic in float64 (autograd supplies
the exact gradient of the written-out forward), following the paper
(/root/reference/PAPER.md, cited ``P:<line>``) and, where the paper is silent,
the readings R1..R20 recorded in DESIGN.md §3 (BigGAN / SNGAN conventions the
paper cites at P:56).

Pins (tests/test_oracle_*.py, all ``-m "not gpu"``):
  * bf16 RNE       -> independent bit formula over every sign/exponent/mantissa-high
                      pattern (P:202 bf16 storage)
  * layout pack    -> brute-force index loops, round trip, P:239 padding example
  * spectral norm  -> numpy SVD sigma_max, rank-1 closed form, monotone bound
  * conv / pools   -> brute-force loops, adjoint identity, delta kernels
  * BN / CBN       -> mean 0 / var 1, sum(dx)=0, split-batch statistics identity
  * hinge          -> closed forms at logits 0 and for a perfect D
  * Adam           -> first step = -lr*g/(|g|+eps), independent scalar loop
  * full step      -> central finite differences on micro nets (fp64)
  * architecture   -> 158,416,358 parameters = "158.42M" (Table 1)
"""

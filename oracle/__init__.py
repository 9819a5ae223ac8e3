"""TEST INFRASTRUCTURE: CPU oracle (restatement of the reference engine).

Never imported by the product package.  See oracle/gt_oracle.c.
"""

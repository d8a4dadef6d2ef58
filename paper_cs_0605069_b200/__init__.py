"""paper_cs_0605069_b200 -- B200-native batched BP decoding of MacKay-Neal codes over GF(2^p).

The product is libgfq.so (CUDA for sm_100a behind the C ABI in include/gfq.h);
this package holds its sources (csrc/), the in-tree build (build.py) and the thin
ctypes binding (gfq.py).  See DESIGN.md.
"""
from . import gfq  # noqa: F401
from .gfq import (GFQ_BEC, GFQ_BIAWGN, GFQ_BSC, GFQ_PUS, GFQ_SUS, Code, Params,  # noqa: F401
                  gfq_decode, gfq_decode_evidence, gfq_decode_host, gfq_decode_stats,
                  gfq_export_messages, gfq_workspace_bytes, gfq_workspace_bytes_host)

"""B200-native row-wise 4-bit clip-search + pack (arXiv 1911.02079 hot path).

Drop-in for the reference package's quantize entry points (``embquant``:
methods.quantize_table / row_clip_range, clipping.clip_range_asym /
clip_range_greedy, histclip.hist_brute_search, packed.pack_table4), computed
by hand-written sm_100a kernels in libeq4.so (C ABI: include/eq4.h).
"""

from ._lib import EXPORTS, Eq4Error, LIB_PATH, load  # noqa: F401
from .api import (  # noqa: F401
    ALL_METHODS,
    AUX_PRECISIONS,
    CODEBOOK_METHODS,
    GPU_METHODS,
    UNIFORM_METHODS,
    ClipRange,
    EmbeddingTable,
    HistWindow,
    PackedTable4,
    RowResults,
    UniformQuantTable,
    WorkCounters,
    clip_range_aciq,
    clip_range_asym,
    clip_range_greedy,
    clip_range_gss,
    clip_range_hist_apprx,
    clip_range_sym,
    clip_range_table,
    clip_range_hist_brute,
    hist_apprx_search,
    hist_brute_search,
    pack_table4,
    packed_row_stride,
    quant_mse,
    quant_mse_rows,
    quantize_pack_table4,
    quantize_table,
    row_clip_range,
)
from .codec import (Histogram, UniformRowQuant, bin_l2_norm, build_histogram,  # noqa: F401
                    dequantize_uniform, quantize_table_uniform, quantize_uniform, unpack_row,
                    unpack_row_codes)
from .codebook import (CodebookQuantTable, CodebookRowQuant, quantize_row_kmeans,  # noqa: F401
                       quantize_table_kmeans)
from .pooled import PooledQuery, bytes_per_pooled_row, sparse_lengths_sum_4bit  # noqa: F401
from .fileio import (DataError, quantize_file, read_embq, read_embt, write_embq,  # noqa: F401
                     write_embt)

__version__ = "0.1.0"

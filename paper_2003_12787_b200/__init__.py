"""B200-native linear ADER-DG Space-Time Predictor (STP).

The product is ``libaderstp.so`` (sm_100a CUDA kernels behind the C ABI declared in
``include/aderstp.h``).  This package is the thin Python host mirror of the reference's
predictor interface (``/root/reference/proj/include/ader/predictor.hpp``), used by the tests and
``bench.py``; PyTorch only provides device memory and streams.  There is no CPU fallback: if the
CUDA library is missing, importing the kernels raises.
"""
from .stp import (  # noqa: F401
    ADERSTP_ERR_CUDA,
    ADERSTP_ERR_INVALID_ARG,
    ADERSTP_ERR_MATERIAL,
    ADERSTP_ERR_NONFINITE,
    ADERSTP_ERR_UNSUPPORTED,
    LAYOUT_AOS,
    LAYOUT_AOSOA,
    PAR_LAMBDA_MU_RHO,
    PAR_RHO_CP_CS,
    AdvectionPde,
    BasisOperators,
    DemoPde,
    ElasticPde,
    LinearPde,
    NcpAdvectionPde,
    Plan,
    PointSourceSpec,
    PredictorOutput,
    SourceOnlyPde,
    StpError,
    advection_pde,
    byte_count,
    convert_layout,
    elastic_pde,
    flop_count,
    generate,
    lib,
    library_path,
    linear_pde,
    make_basis,
    ncp_advection_pde,
    paper_demo_pde,
    predict,
    source_only_pde,
    stable_dt,
)

__all__ = [name for name in dir() if not name.startswith("_")]

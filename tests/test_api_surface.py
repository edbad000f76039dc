"""The drop-in surface: every name the reference package exports
(pkg/src/bzc/__init__.py:12-63, and the public names of ops.py / metrics.py /
codec.py) is an attribute of paper_2406_11209_b200.  Parsed from a frozen
list (the reference tree does not travel to the GPU box)."""

import paper_2406_11209_b200 as bz

# pkg/src/bzc/__init__.py:12-63, in file order
REFERENCE_EXPORTS = [
    "BlockedArray", "DenseArray", "block", "convert_precision", "gradient_array", "unblock",
    "CodecSettings", "CompressedArray", "PruningMask", "bin_coefficients", "compress",
    "decompress", "prune_and_flatten", "specified_coefficients", "unflatten",
    "BzcError",
    "bitstream_layout", "deserialize", "serialize",
    "FloatKind", "IndexKind",
    "compare_against_oracle", "compression_ratio", "measure_roundtrip", "measured_ratio",
    "predict_error_bounds",
    "SsimParams", "WassersteinParams", "add", "add_scalar", "approx_wasserstein",
    "cosine_similarity", "covariance", "dot", "l2_norm", "mean", "mul_scalar", "negate", "ssim",
    "variance",
    "TransformFamily", "TransformMatrix", "forward_transform", "inverse_transform",
    "make_transform",
    "__version__",
]

# metrics.py:35-47 __all__
METRICS_ALL = ["compression_ratio", "measured_ratio", "RatioReport", "ratio_report",
               "ErrorReport", "predict_error_bounds", "measure_roundtrip", "OpComparison",
               "compare_against_oracle", "ORACLE_OPERATIONS", "render_table", "render_records"]

# errors.py:29-90
ERRORS = ["BzcError", "DimensionMismatch", "NonPowerOfTwoBlock", "DegenerateShape",
          "LengthMismatch", "IndexRangeError", "SettingsMismatch", "MaskExcludesMeanCoefficient",
          "ZeroNormOperand", "NegativeBaseWithFractionalWeight", "UnknownOperation",
          "FormatError", "TruncatedStream", "InvalidTypeCode", "ZeroExtent", "ArrayFileError"]


def test_every_reference_export_is_present():
    missing = [n for n in REFERENCE_EXPORTS if not hasattr(bz, n)]
    assert not missing, missing


def test_metrics_module_surface():
    from paper_2406_11209_b200 import metrics

    missing = [n for n in METRICS_ALL if not hasattr(metrics, n)]
    assert not missing, missing
    assert metrics.ORACLE_OPERATIONS == {
        "dot": (2, "scalar"), "mean": (1, "scalar"), "covariance": (2, "scalar"),
        "variance": (1, "scalar"), "l2_norm": (1, "scalar"),
        "cosine_similarity": (2, "scalar"), "ssim": (2, "scalar"),
        "wasserstein": (2, "scalar"), "negate": (1, "array"), "add": (2, "array"),
        "add_scalar": (1, "array"), "mul_scalar": (1, "array")}


def test_error_hierarchy():
    from paper_2406_11209_b200 import errors

    for n in ERRORS:
        cls = getattr(errors, n)
        assert issubclass(cls, errors.BzcError)
    assert issubclass(errors.TruncatedStream, errors.FormatError)


def test_compare_against_oracle_validates_before_compute():
    """metrics.py:244-250: unknown names and wrong arity raise before any GPU work."""
    import pytest

    from paper_2406_11209_b200 import errors, metrics

    s = bz.CodecSettings((4, 4))
    with pytest.raises(errors.UnknownOperation):
        metrics.compare_against_oracle("median", [], s)
    with pytest.raises(ValueError, match="takes 2 operand"):
        metrics.compare_against_oracle("dot", [object()], s)


def test_renderers_match_reference_format():
    from paper_2406_11209_b200 import metrics

    c = [metrics.OpComparison("dot", "scalar", 1.5, 1.25, 0.25, 0.2),
         metrics.OpComparison("add", "array", None, None, 0.0, 0.0, 0.125, "rebinning")]
    table = metrics.render_table(c).splitlines()
    assert table[0].split() == ["operation", "type", "compressed", "oracle", "abs_deviation",
                                "rel_deviation", "bound", "note"]
    assert table[1].split() == ["dot", "scalar", "1.5", "1.25", "0.25", "0.20000000000000001",
                                "-", "-"]
    rec = metrics.render_records(c).split("\n\n")
    assert rec[1].splitlines() == ["operation=add", "result_type=array", "compressed=-",
                                   "oracle=-", "absolute_deviation=0", "relative_deviation=0",
                                   "bound=0.125", "note=rebinning"]

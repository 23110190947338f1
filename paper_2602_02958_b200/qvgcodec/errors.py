"""Exception classes of the drop-in API (mirrors Q/errors.py:8-73).

Same names and bases as the reference so ``except CodecError`` /
``except ValueError`` clauses written against ``qvgcodec`` keep working.
"""


class CodecError(Exception):
    """Root of every codec failure."""


def _value_error(name: str, doc: str):
    return type(name, (CodecError, ValueError), {"__doc__": doc})


DimensionMismatch = _value_error("DimensionMismatch", "Shape / divisibility constraint violated.")
NonFiniteInput = _value_error("NonFiniteInput", "NaN or Inf in an input tensor.")
EmptyPlane = _value_error("EmptyPlane", "Plane with no tokens or no channels.")
EmptyInput = _value_error("EmptyInput", "Clustering called on zero rows.")
NonFiniteScale = _value_error("NonFiniteScale", "Scale is NaN/Inf and has no E4M3 code.")
NaNPattern = _value_error("NaNPattern", "E4M3 byte 0x7F / 0xFF (NaN pattern).")
RangeOverflow = _value_error("RangeOverflow", "Integer code outside the symmetric b-bit range.")
Truncated = _value_error("Truncated", "Byte stream shorter than its declared contents.")
BadMagic = _value_error("BadMagic", "Missing file magic.")
UnknownDtype = _value_error("UnknownDtype", "Unsupported raw-tensor dtype code.")
BadParams = _value_error("BadParams", "Parameter outside its domain.")
NotPowerOfTwo = _value_error("NotPowerOfTwo", "Length is not a power of two.")
ShapeMismatch = _value_error("ShapeMismatch", "Two operands disagree in shape.")
ConfigMismatch = _value_error("ConfigMismatch", "Chunk config disagrees with its header.")
CorruptChunk = _value_error("CorruptChunk", "Chunk record failed validation.")
# raised by this implementation only: a shape the sm_100a kernels do not cover
UnsupportedShape = _value_error("UnsupportedShape", "Shape outside the compiled kernels.")


class OutOfRange(CodecError, IndexError):
    """Chunk index outside the valid range."""


for _c in (DimensionMismatch, NonFiniteInput, EmptyPlane, EmptyInput, NonFiniteScale, NaNPattern,
           RangeOverflow, Truncated, BadMagic, UnknownDtype, BadParams, NotPowerOfTwo,
           ShapeMismatch, ConfigMismatch, CorruptChunk, UnsupportedShape):
    _c.__module__ = __name__
del _c

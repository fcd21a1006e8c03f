"""Exception hierarchy, name-compatible with the reference (errors.py:1-60).

Callers that catch the reference's exception classes by name keep working:
every class below has the reference's name and parent.  ``ExecutionError``
additionally covers a missing native library and CUDA failures, which the
reference cannot raise.
"""


class VoxplanError(Exception):
    pass


class ModelError(VoxplanError):
    pass


class ParseError(ModelError):
    """Carries the 1-based source position of a prototxt syntax error."""

    def __init__(self, message, line=None, column=None):
        self.line, self.column = line, column
        super().__init__(message if line is None else "line %d: %s" % (line, message))


def _subclass(name, parent):
    return type(name, (parent,), {"__module__": __name__})


LayoutError = _subclass("LayoutError", VoxplanError)
FormatError = _subclass("FormatError", VoxplanError)
PlanError = _subclass("PlanError", VoxplanError)
ExecutionError = _subclass("ExecutionError", VoxplanError)
TileError = _subclass("TileError", VoxplanError)
UnknownLayerError = _subclass("UnknownLayerError", ModelError)
DanglingReferenceError = _subclass("DanglingReferenceError", ModelError)
DuplicateTopError = _subclass("DuplicateTopError", ModelError)
CycleError = _subclass("CycleError", ModelError)
ShapeError = _subclass("ShapeError", ModelError)

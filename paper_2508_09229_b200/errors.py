"""Error classes of the ``moeplace`` API (same names and hierarchy as the reference package,
/root/reference/pkg/src/moeplace/errors.py:8-31), plus the CLI exit-code table
(errors.py:3-4 and SPEC.md:436: 2 = configuration, 3 = infeasible, 4 = io/parse)."""

EXIT_OK = 0
EXIT_CONFIG = 2
EXIT_INFEASIBLE = 3
EXIT_PARSE = 4


class MoeplaceError(Exception):
    """Root of every error this package raises."""


class ConfigError(MoeplaceError):
    """A configuration or argument value is invalid (bad value, unknown key, bad combination)."""


class TopologyError(MoeplaceError):
    """The cluster graph is malformed, e.g. not connected."""


class TraceParseError(MoeplaceError):
    """An activation-trace file could not be parsed; ``line_no`` is 1-based when known."""

    def __init__(self, message, line_no=None):
        self.line_no = line_no
        super().__init__(message if line_no is None else "line %d: %s" % (line_no, message))


class InfeasibleError(MoeplaceError):
    """The capacity constraints admit no placement."""


def exit_code(exc: BaseException) -> int:
    """CLI exit code for an exception."""
    if isinstance(exc, InfeasibleError):
        return EXIT_INFEASIBLE
    if isinstance(exc, (TraceParseError, OSError)):
        return EXIT_PARSE
    if isinstance(exc, MoeplaceError):
        return EXIT_CONFIG
    return 1

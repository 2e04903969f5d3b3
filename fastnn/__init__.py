"""`import fastnn` compatibility shim: the reference package name, served by the
B200-native build in paper_2503_10017_b200 (see that package's docstring)."""
from paper_2503_10017_b200 import *  # noqa: F401,F403
from paper_2503_10017_b200 import __all__, __version__  # noqa: F401

"""The name `orcasim` bound to paper_2008_11578_b200: lets the reference's unmodified test-suite
(staged by __graft_entry__.install_reference into the git-ignored baseline/_ref/_tests) run against
the GPU package -- tests/test_gpu_refsuite.py. Test infrastructure only."""
from paper_2008_11578_b200 import *  # noqa: F401,F403
from paper_2008_11578_b200 import __all__  # noqa: F401

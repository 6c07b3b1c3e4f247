"""`orcasim.scenario` as the reference's own tests import it, served by paper_2008_11578_b200
(tests/test_gpu_refsuite.py). Test infrastructure: a re-export, no logic."""
import paper_2008_11578_b200.scenario as _m
globals().update({k: v for k, v in vars(_m).items() if not k.startswith('__')})

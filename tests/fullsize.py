"""Session cache of the BASELINE full-size synthetic problems (c3-c5 take 5 s to ~3 min
to render), shared by the full-size GPU tests.  The returned Problem must not be mutated."""
import functools

import synth


@functools.lru_cache(maxsize=None)
def full_config(k: int):
    return synth.make_config(k)

"""Reaction correction M_R x on the device (assembly.py:287-347)."""


def set_reaction(ctx, st, final_time, consts, u, w, lengths):
    raise NotImplementedError("reaction correction kernel not built yet")

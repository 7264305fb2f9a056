"""Picklable engine factory for the spawned par_eliminate workers in the CPU
tests: each worker rank runs the C oracle (test infrastructure) instead of a
device context, so the fork / rendezvous / broadcast / reassembly logic of
parexec._spawn_run runs without a GPU."""


def make(n, p, kind, rank, world):
    import oracle
    return oracle.OracleRank(n, p, kind, rank, world, 1)

"""Reader of the paper-printed fixtures under tests/golden/ (each file cites its passage)."""
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def table1():
    """{(problem, tolerance): average Jacobi iterations} from PAPER.md:575-594 (Table 1)."""
    out = {}
    with open(os.path.join(GOLDEN, "table1_jacobi_iters.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            prob, tol, avg = line.split()
            out[(prob, float(tol))] = float(avg)
    return out

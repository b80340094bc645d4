"""One training step out of an ncu launch list of bench.py (the kernels between
two consecutive plan_next launches of the graph-replayed timed region).

python tools/ncu_step_breakdown.py launches.csv [which=-2]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from ncu_summary import load  # noqa: E402


def main(path, which=-2):
    rows = load(path)
    starts = [i for i, (_, name, _) in enumerate(rows) if "plan_next_kernel" in name]
    # training steps only: intervals that contain the optimizer (the bench's prep-only
    # passes also launch plan_next)
    steps = [(a, b) for a, b in zip(starts, starts[1:])
             if any("adam_kernel" in n for _, n, _ in rows[a:b])]
    a, b = steps[which]
    step = rows[a:b]
    tot = sum(us for _, _, us in step)
    for _, name, us in step:
        print(f"{us:8.1f} us  {name.split('(')[0].replace('void ', '')[:100]}")
    print(f"total {tot:.1f} us serialised over {len(step)} launches "
          f"(ncu: cold caches, no prep/compute overlap — compare shares, not absolutes)")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else -2)

from paper_2411_17089_b200.cli import *  # noqa: F401,F403
from paper_2411_17089_b200 import cli as _m

globals().update({k: v for k, v in vars(_m).items() if not k.startswith("__")})

if __name__ == "__main__":  # python -m kvoverlap.cli
    raise SystemExit(_m.main())

from paper_2411_17089_b200.costmodel import *  # noqa: F401,F403
from paper_2411_17089_b200 import costmodel as _m

globals().update({k: v for k, v in vars(_m).items() if not k.startswith("__")})

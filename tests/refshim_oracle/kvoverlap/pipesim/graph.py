from paper_2411_17089_b200 import pipesim as _m

globals().update({k: v for k, v in vars(_m).items() if not k.startswith("__")})

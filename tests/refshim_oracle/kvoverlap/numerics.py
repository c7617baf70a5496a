from oracle import numerics_ref as _m

globals().update({k: v for k, v in vars(_m).items() if not k.startswith("__")})

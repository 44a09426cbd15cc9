from .scenes import *

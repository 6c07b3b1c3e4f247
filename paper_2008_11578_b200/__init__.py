"""B200-native ORCA steering step (arXiv 2008.11578) behind the reference's
public simulation API. See DESIGN.md."""

from .types import (AgentClass, ClassParams, FrameMetrics, ResponsibilityMatrix,
                    ScenarioConfig, SimState)

__all__ = ["AgentClass", "ClassParams", "FrameMetrics", "ResponsibilityMatrix",
           "ScenarioConfig", "SimState"]
